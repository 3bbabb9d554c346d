#!/usr/bin/env bash
# Install the UNMODIFIED reference (sliceprop 0.1.0 + the pysliceprop
# binding, /root/reference/pkg) into baseline/_ref (git-ignored, travels to
# the GPU box with gpurun) and stage its own test suites next to it, so that
#   - bench.py times the real reference on the box's host cores, and
#   - tests/test_reference_suites.py runs the reference's tests against the
#     drop-in (aliasing `sliceprop` / `pysliceprop` to this package).
# Nothing here is tracked by git; /root/reference is read-only, so the build
# runs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d /tmp/refpkg.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$DST"
mkdir -p "$DST"
PIP=(python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse
     --no-deps --target "$DST")
"${PIP[@]}" "$TMP" >/dev/null
"${PIP[@]}" "$TMP/bindings" >/dev/null
# the reference's own test suites, verbatim
mkdir -p "$DST/ref_tests/core" "$DST/ref_tests/bindings"
cp "$TMP"/tests/*.py "$DST/ref_tests/core/"
cp "$TMP"/bindings/tests/*.py "$DST/ref_tests/bindings/"
rm -rf "$TMP"
python - "$DST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import sliceprop, pysliceprop
print("installed", sliceprop.__file__, pysliceprop.__file__)
PY
