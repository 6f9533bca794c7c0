#!/bin/bash
# Install the UNMODIFIED reference package (pure-Python ssimkit) into baseline/_ref for
# bench.py --impl reference and the cpu_baseline leg.  baseline/_ref is git-ignored (not
# product source) but not gpurun-ignored, so it travels to the GPU box with the snapshot.
# The build writes into its source tree, so it installs from a copy under /tmp
# (/root/reference is read-only); numpy and click are already in the image (--no-deps).
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
# the reference's own test files, run against the engine by tests/test_gpu_reference_suite.py
# (through the ssimkit alias in tests/refsuite; they stay untracked like the package itself)
cp -r "$SRC/tests" "$REPO/baseline/_ref/ssimkit_tests"
python -c "import sys; sys.path.insert(0, '$REPO/baseline/_ref'); import ssimkit; print('ssimkit', ssimkit.__file__)"
