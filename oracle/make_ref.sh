#!/usr/bin/env bash
# Stage the reference package and its own test suite into oracle/_ref/
# (git-ignored; it travels to the GPU box with the gpurun snapshot) so that
# tests/test_reference_suite_gpu.py can run the reference's tests unchanged
# against the GPU index and engine.  TEST INFRASTRUCTURE ONLY: nothing in
# paper_2509_17360_b200/ reads oracle/.  The reference is pure Python, so
# "building" it is a copy of pkg/src/semcache and pkg/tests.
set -euo pipefail
REF=${1:-/root/reference}
HERE=$(cd "$(dirname "$0")" && pwd)
OUT="$HERE/_ref"
if [ ! -d "$REF/pkg/src/semcache" ]; then
    echo "make_ref: $REF/pkg/src/semcache not found; oracle/_ref left as is" >&2
    exit 0
fi
rm -rf "$OUT.tmp"
mkdir -p "$OUT.tmp"
cp -r "$REF/pkg/src/semcache" "$OUT.tmp/semcache"
cp -r "$REF/pkg/tests" "$OUT.tmp/tests"
find "$OUT.tmp" -name __pycache__ -prune -exec rm -rf {} +
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
echo "make_ref: staged semcache + tests into $OUT"
