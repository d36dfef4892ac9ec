#!/bin/bash
# Install the UNMODIFIED reference package (pkg/, pure Python + numpy) into
# baseline/_ref for bench.py's reference arm and cpu_baseline leg.  Run in the
# build container (where /root/reference exists); baseline/_ref is git-ignored
# but travels to the GPU box with gpurun.  The build writes into its source
# tree, so it installs from a copy under /tmp (/root/reference is read-only).
set -euo pipefail
cd "$(dirname "$0")/.."
rm -rf /tmp/lfps_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/lfps_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/lfps_ref_src
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import lfps; print('reference lfps', lfps.__file__)"
# the reference's own test suite, for tests/test_gpu_reference_suite.py (run
# against this package with `lfps` aliased to paper_2506_15704_b200.lfps)
rm -rf baseline/_ref_tests
cp -r /root/reference/pkg/tests baseline/_ref_tests
echo "reference tests copied to baseline/_ref_tests"
