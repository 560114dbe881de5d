#!/bin/sh
# Install the UNMODIFIED reference into baseline/_ref (git-ignored, not gpurun-ignored:
# it travels to the GPU box).  /root/reference is read-only, so the build runs from a
# copy under /tmp.  The reference's own table tests are staged next to it for
# tests/test_gpu_dropin.py (they are not part of this repo).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/pf_refsrc baseline/_ref
cp -r /root/reference/pkg /tmp/pf_refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/pf_refsrc
mkdir -p baseline/_ref/_ref_tests
cp /root/reference/pkg/tests/test_table.py /root/reference/pkg/tests/conftest.py \
    baseline/_ref/_ref_tests/
