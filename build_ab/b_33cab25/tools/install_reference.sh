#!/usr/bin/env bash
# Install the UNMODIFIED reference (sketchlpa 0.1.0) into baseline/_ref
# (git-ignored; travels to the GPU box with the gpurun snapshot) and put its
# own test-suite and docs beside it, for tests/test_reference_suite.py (the
# reference's tests run against the drop-in) and bench.py --impl reference
# (the Python reference timed on the box's host).  Build-container only:
# /root/reference does not exist on the GPU box.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
mkdir -p "$REPO/baseline/_ref/sketchlpa_suite"
cp -r "$SRC/tests" "$SRC/docs" "$REPO/baseline/_ref/sketchlpa_suite/"
rm -rf "$TMP"
echo "installed: $(ls "$REPO/baseline/_ref")"
