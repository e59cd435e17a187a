#!/bin/bash
# Stage the reference's own test modules for the QMCUR path next to the installed reference
# (baseline/_ref is git-ignored and travels to the GPU box; the sources are never committed).
# tests/test_gpu_reference_suite.py runs them against this repository's GPU implementation
# through the import shim tests/ref_shim/qcur.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg/tests
DST=$ROOT/baseline/_ref/tests_ref
[ -d "$SRC" ] || { echo "no reference tests at $SRC"; exit 0; }
mkdir -p "$DST"
for f in conftest.py helpers.py test_cur.py test_linalg.py test_quat.py test_completion.py; do
  cp "$SRC/$f" "$DST/$f"
done
[ -d "$SRC/data" ] && cp -r "$SRC/data" "$DST/" || true
echo "staged $(ls "$DST" | wc -l) files in $DST"
