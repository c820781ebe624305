#!/bin/bash
# Install the UNMODIFIED reference (efgraph 0.1.0, /root/reference/pkg) into the
# git-ignored baseline/_ref/ so it travels to the GPU box with gpurun.
#  * the package: pip --target from a copy under /tmp (the source tree is
#    read-only); --no-deps because numpy is already in the image and the
#    wheelhouse has no numpy wheel (resolution fails otherwise);
#  * its test suite (pkg/tests, not part of the wheel) beside it as
#    baseline/_ref/efgraph_tests/, so tests/test_gpu_reference_suite.py can run
#    the reference's own EF tests against the GPU backend on the box.
# Nothing here is committed: baseline/_ref/ is in .gitignore.
set -euo pipefail
cd "$(dirname "$0")/.."
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "reference not found at $SRC"; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$TMP/pkg" > /dev/null
cp -r "$SRC/tests" baseline/_ref/efgraph_tests
rm -rf "$TMP"
python - <<'P'
import sys; sys.path.insert(0, "baseline/_ref")
import efgraph; print("installed efgraph", efgraph.__version__, "->", efgraph.__file__)
P
