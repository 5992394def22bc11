#!/bin/bash
# Install the UNMODIFIED reference package (`hinm`, /root/reference/pkg) into oracle/_ref so that
# the CPU arms of bench.py (--impl reference, cpu_baseline) and the parity tooling can run the
# reference's own code on the GPU box, where /root/reference does not exist.  Test/measurement
# infrastructure only: the product package never imports it.  oracle/_ref is git-ignored (the
# reference's sources stay out of this repo's history) but travels with the gpurun snapshot.
#
#   bash oracle/install_ref.sh            # no network: offline wheelhouse, no dependency resolution
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${HINM_REFERENCE:-/root/reference/pkg}"
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "install_ref: $SRC not found (reference checkout absent); nothing to do" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"                  # the build writes egg-info: never into the read-only tree
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
PYTHONPATH="$HERE/_ref" python -c "import hinm; print('install_ref: hinm', hinm.__file__)"
