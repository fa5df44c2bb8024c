#!/bin/sh
# Install the UNMODIFIED reference package (pure Python + numba) into
# baseline/_ref (git-ignored; it travels to the GPU box with the gpurun
# snapshot).  The source tree is read-only, so the build runs from a copy.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import rangeseg; print('reference', rangeseg.__version__, 'in', '$HERE/_ref')"
