#!/usr/bin/env bash
# One-time offline install of the UNMODIFIED reference into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot):
#   * the `groupnb` package, pip-installed from a /tmp copy of
#     /root/reference/pkg (the source tree is read-only);
#   * the reference's own test suite (pkg/tests) next to it, so
#     tests/test_reference_suite.py can run it with the GPU backend installed.
# Nothing from the reference is committed to this repository.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
echo "installed groupnb + its tests into $ROOT/baseline/_ref"
