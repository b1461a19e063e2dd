#!/usr/bin/env bash
# Install the UNMODIFIED reference package (fiberdbp, pure Python) into
# oracle/_ref so bench.py's reference arm and cpu_baseline can time the
# reference's own backpropagate (pkg/src/fiberdbp/dbp.py:160) on the GPU box,
# where /root/reference does not exist.  oracle/_ref is git-ignored but not
# gpurun-ignored, so it travels with the snapshot.  The build writes into its
# source tree, hence the copy under /tmp; dependencies (numpy, scipy, numba)
# are already in the image, hence --no-deps.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${FIBERDBP_SRC:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference source $SRC not found" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/oracle/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/oracle/_ref" "$TMP/pkg"
echo "installed fiberdbp into $REPO/oracle/_ref"
