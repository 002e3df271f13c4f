#!/bin/bash
# Install the UNMODIFIED reference (splatsort, pure Python) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot).  The
# reference's own tests are copied next to it so tests/test_reference_replay.py
# can replay them through the B200 path on the box (/root/reference does not
# exist there).  Offline: --no-index from the image wheelhouse; --no-deps
# because numpy / scipy / pillow are already in the image.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"                      # the build writes into the tree
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$HERE/_ref/tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import splatsort; print('splatsort', splatsort.__file__)"
