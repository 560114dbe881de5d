#!/bin/bash
# Build the working tree's library with extra nvcc flags as tools/_var/<name>.so
# usage: bash tools/build_variant.sh <name> -DFLAG=VALUE ...
set -e
name=$1; shift
mkdir -p tools/_var
python - "$name" "$@" <<'PY'
import subprocess, sys
sys.path.insert(0, '.')
from paper_1902_05942_b200 import _lib
name, extra = sys.argv[1], sys.argv[2:]
subprocess.check_call(['nvcc', *_lib.NVCC_FLAGS, *extra, '-o', f'tools/_var/{name}.so', *_lib.SOURCES])
PY
