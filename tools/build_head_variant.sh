#!/bin/bash
# Build the committed HEAD's library as tools/_var/head.so (A/B against the working tree
# in one gpurun call: bash tools/bench_variants.sh base head)
set -e
tmp=$(mktemp -d)
git archive HEAD paper_1902_05942_b200/csrc include | tar -x -C "$tmp"
mkdir -p tools/_var
python - "$tmp" <<'PY'
import subprocess, sys, os
sys.path.insert(0, '.')
from paper_1902_05942_b200 import _lib
tmp = sys.argv[1]
srcs = [os.path.join(tmp, os.path.relpath(s, '.')) for s in _lib.SOURCES]
subprocess.check_call(['nvcc', *_lib.NVCC_FLAGS, '-o', 'tools/_var/head.so', *srcs])
PY
rm -rf "$tmp"
