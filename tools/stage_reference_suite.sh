#!/bin/sh
# Stage the reference's own test files + sources (read-only inputs, not
# product code) into the git-ignored baseline/_ref_suite/, so that
# tests/test_reference_suite_gpu.py can run them on the GPU box against the
# drop-in (the box has no /root/reference; the staged copy travels with the
# gpurun snapshot like baseline/_ref).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${1:-/root/reference/pkg}
DST="$ROOT/baseline/_ref_suite"
rm -rf "$DST"
mkdir -p "$DST/pkg" "$DST/bindings"
cp -r "$REF/tests" "$DST/tests"
cp -r "$REF/src/spatialhash" "$DST/pkg/spatialhash"
cp -r "$REF/bindings/tests" "$DST/bindings_tests"
cp -r "$REF/bindings/src/spatialhash_arrays" "$DST/bindings/spatialhash_arrays"
find "$DST" -name __pycache__ -prune -exec rm -rf {} +
echo "staged into $DST"
