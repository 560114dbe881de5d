#!/bin/bash
# Build the library of a given commit as tools/_var/<name>.so (bisecting with bench_variants.sh)
# usage: bash tools/build_commit_variant.sh <name> <commit>
set -e
name=$1; rev=$2
tmp=$(mktemp -d)
git archive "$rev" paper_1902_05942_b200/csrc include | tar -x -C "$tmp"
mkdir -p tools/_var
python - "$tmp" "$name" <<'PY'
import subprocess, sys, os
sys.path.insert(0, '.')
from paper_1902_05942_b200 import _lib
tmp, name = sys.argv[1], sys.argv[2]
srcs = [os.path.join(tmp, os.path.relpath(s, '.')) for s in _lib.SOURCES]
subprocess.check_call(['nvcc', *_lib.NVCC_FLAGS, '-o', f'tools/_var/{name}.so', *srcs])
PY
rm -rf "$tmp"
