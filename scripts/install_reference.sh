#!/bin/bash
# One-time offline install of the UNMODIFIED reference (covault) into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun): the reference arm of bench.py and the exception types the
# drop-in shares.  Also stages the reference's own test suites and scenario assets under
# baseline/_ref/ref_pkg/ so tests/test_reference_suites_gpu.py can run them against the GPU path
# on a box where /root/reference does not exist.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$REF" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg" > /dev/null
rm -rf "$ROOT/baseline/_ref/ref_pkg"
mkdir -p "$ROOT/baseline/_ref/ref_pkg"
cp -r "$REF/tests" "$REF/scenarios" "$ROOT/baseline/_ref/ref_pkg/"
rm -rf "$TMP"
echo "reference installed into $ROOT/baseline/_ref (tests staged in ref_pkg/)"
