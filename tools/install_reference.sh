#!/usr/bin/env bash
# Install the UNMODIFIED reference package (duetsim, pure NumPy) into
# baseline/_ref for bench.py's reference arm and CPU baseline.  Run in the
# build container (the only place /root/reference exists); baseline/_ref is
# git-ignored but not gpurun-ignored, so it travels to the GPU box.
# The build writes into its source tree, so it installs from a /tmp copy;
# numpy/scipy are already in the image (--no-deps: no index is reachable).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
(cd /tmp && PYTHONPATH="$ROOT/baseline/_ref" python -c "import duetsim; print('reference installed:', duetsim.__file__)")
