#!/bin/sh
# Install the UNMODIFIED reference (tissuemix, pure Python) into baseline/_ref -- git-ignored,
# not gpurun-ignored, so it travels to the GPU box -- together with its own test suite, which
# tests/test_gpu_reference_suite_live.py runs against the drop-in (vb.install()) on a B200.
# The build writes into its source tree, so it installs from a copy under /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${REFERENCE:-/root/reference}
rm -rf /tmp/tissuemix_src "$ROOT/baseline/_ref"
cp -r "$SRC/pkg" /tmp/tissuemix_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/tissuemix_src
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/tests"
echo "reference installed into $ROOT/baseline/_ref (package + tests)"
