#!/usr/bin/env bash
# Install the unmodified reference (pcbz, /root/reference/pkg) into
# baseline/_ref (git-ignored, travels to the GPU box with gpurun) from the
# offline wheelhouse, and stage its own test suite next to it
# (baseline/_ref/pcbz_tests) so tests/test_reference_suite.py can run the
# reference's tests against the B200 path where /root/reference is absent.
set -euo pipefail
cd "$(dirname "$0")/.."
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$TMP/pkg"
cp -r "$SRC/tests" baseline/_ref/pcbz_tests
rm -rf "$TMP" baseline/_ref/pcbz_tests/__pycache__
echo "installed $(ls baseline/_ref)"
