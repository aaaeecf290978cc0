#!/usr/bin/env bash
# Install the unmodified reference (tomokit + tomokit_layers) into baseline/_ref
# (git-ignored, travels to the GPU box with gpurun), plus a copy of its own test
# suites under baseline/_ref/ref_tests/ for scripts/run_reference_suite.py.
# Offline: --no-index from the local wheelhouse; the sources are copied to /tmp
# first because the build writes into the source tree (/root/reference is read-only).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${1:-/root/reference}"
rm -rf /tmp/tk_refcopy "$ROOT/baseline/_ref"
cp -r "$REF/pkg" /tmp/tk_refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/tk_refcopy /tmp/tk_refcopy/bindings
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/ref_tests/pkg_tests"
cp -r "$REF/pkg/bindings/tests" "$ROOT/baseline/_ref/ref_tests/bindings_tests"
cp -r "$REF/pkg/configs" "$ROOT/baseline/_ref/ref_tests/configs" 2>/dev/null || true
# test_acceptance.py criterion 7 runs pkg/scripts/artifact_gallery.py relative to its own directory
cp -r "$REF/pkg/scripts" "$ROOT/baseline/_ref/ref_tests/scripts" 2>/dev/null || true
echo "installed tomokit into $ROOT/baseline/_ref"
