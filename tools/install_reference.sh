#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) -- the one offline install the task
# allows -- plus a copy of its own test files under baseline/_ref/multilap_tests
# so tests/test_reference_suite.py can run the reference's tests against the
# INTEGRATION.md shim on the GPU box (where /root/reference does not exist).
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${MULTILAP_SRC:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; /root/reference is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" -q
rm -rf "$ROOT/baseline/_ref/multilap_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/multilap_tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import multilap; print('multilap', multilap.__file__)"
