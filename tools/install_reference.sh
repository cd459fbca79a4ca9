#!/bin/bash
# Install the UNMODIFIED reference package (pure Python + NumPy, /root/reference/pkg)
# into baseline/_ref for bench.py --impl reference.  /root/reference is read-only,
# so the build runs from a copy under /tmp.  baseline/_ref is git-ignored and
# travels to the GPU box with the gpurun snapshot.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import dhsa; print('reference installed:', dhsa.__file__)"
