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
