#!/bin/bash
# Install the UNMODIFIED reference (semsplat, pure Python) into baseline/_ref
# (git-ignored, travels to the GPU box with the gpurun snapshot) together with
# a copy of its own test directory, which tests/test_reference_suite_gpu.py runs
# against the B200 path through paper_2603_09632_b200.reference_shim.
# Run in the build container (where /root/reference exists).
set -euo pipefail
cd "$(dirname "$0")/.."
REF=${REF:-/root/reference}
[ -d "$REF/pkg" ] || { echo "no reference at $REF"; exit 1; }
rm -rf /tmp/semsplat_src baseline/_ref
cp -r "$REF/pkg" /tmp/semsplat_src          # the build writes egg-info into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/semsplat_src > /dev/null
cp -r "$REF/pkg/tests" baseline/_ref/semsplat_tests
echo "installed: $(ls baseline/_ref)"
