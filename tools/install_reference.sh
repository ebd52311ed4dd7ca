#!/bin/bash
# Install the unmodified reference (mrsim) into baseline/_ref (git-ignored; it travels to the GPU box with
# gpurun), plus a copy of its test suite for the drop-in test (tests/test_gpu_dropin.py).  Offline:
# --no-index against the image's wheelhouse, --no-deps (numpy and scipy are in the image already; the
# reference pins none of them).  The build writes into its source tree, so it runs from a copy in /tmp.
set -euo pipefail
REF=${1:-/root/reference/pkg}
cd "$(dirname "$0")/.."
rm -rf baseline/_ref /tmp/mrsim_src && cp -r "$REF" /tmp/mrsim_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse --target baseline/_ref /tmp/mrsim_src
mkdir -p baseline/_ref/mrsim_tests && cp "$REF"/tests/*.py baseline/_ref/mrsim_tests/
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import mrsim; print('mrsim', mrsim.__file__)"
