#!/bin/bash
# Install the unmodified reference package into baseline/_ref (git-ignored,
# travels to the GPU box) for tests/test_reference_gate.py.  The build writes
# into the source tree, so it runs from a scratch copy (/root/reference is
# read-only).  The reference's tests/ are staged beside the package.
set -e
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d /tmp/refpkg.XXXXXX)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
mkdir -p "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg" 2>&1 | tail -3
cp -r "$SRC/tests" "$REPO/baseline/_ref/tests"
rm -rf "$TMP"
ls "$REPO/baseline/_ref"
