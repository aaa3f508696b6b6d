#!/bin/bash
# Installs the UNMODIFIED reference (optistate, /root/reference/pkg) into
# baseline/_ref (git-ignored; travels to the GPU box with the gpurun snapshot)
# plus a copy of its own test suite under baseline/_ref/tests.
#   - pip builds in the source tree, and /root/reference is read-only: build from a /tmp copy
#   - the wheelhouse has no numpy/numba wheels (they are already in the image): --no-deps
# Outcome recorded in DESIGN.md §8.
set -euo pipefail
cd "$(dirname "$0")/.."
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/optistate_src"
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref "$TMP/optistate_src"
cp -r "$SRC/tests" baseline/_ref/tests
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import optistate; print('optistate', optistate.__file__)"
