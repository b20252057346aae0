#!/usr/bin/env bash
# Install the unmodified reference (gearserve) into baseline/_ref, the
# git-ignored location the task reserves for it (it travels to the GPU box
# with gpurun snapshots), plus its own test suite, so the reference's tests
# can run against the B200 binding (tests/test_gpu_reference_suite.py).
# Never committed: baseline/_ref/ is in .gitignore.
set -euo pipefail
REF=${1:-/root/reference}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
cp -r "$REF/pkg" "$TMP/pkg"   # the reference tree is read-only; build from a copy
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
  --no-deps --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref"
