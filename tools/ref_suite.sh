#!/usr/bin/env bash
# Run the REFERENCE's own hot-path tests (unmodified) against the drop-in
# `duetsim` shim of this repository.
#
#   tools/ref_suite.sh stage   # in the build container: copy the reference's
#                              # test files into ref_suite/ (git-ignored, not
#                              # gpurun-ignored, so they travel to the GPU box;
#                              # reference sources are never committed)
#   tools/ref_suite.sh run     # on the GPU box: pytest them with `duetsim`
#                              # resolving to ./duetsim (the B200 engine)
#
# Files: the reference's conftest.py + oracles.py (its test oracle) and the
# four hot-path modules test_core / test_statevec / test_fusion /
# test_distsim.  test_circuits / test_cli / test_acceptance import the
# out-of-scope tensor-network modules (duetsim.tn, duetsim.convert) and are
# not staged.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DEST="$ROOT/ref_suite"
case "${1:-run}" in
  stage)
    SRC="${DUETSIM_REF_TESTS:-/root/reference/pkg/tests}"
    rm -rf "$DEST"
    mkdir -p "$DEST"
    for f in conftest.py oracles.py test_core.py test_statevec.py test_fusion.py test_distsim.py; do
      cp "$SRC/$f" "$DEST/$f"
    done
    sha256sum "$DEST"/*.py > "$DEST/SHA256SUMS"
    echo "staged $(ls "$DEST"/test_*.py | wc -l) reference test modules into $DEST"
    ;;
  run)
    cd "$DEST"
    sha256sum -c --quiet SHA256SUMS
    # `duetsim` must resolve to the shim in the repo root, never to a reference copy
    PYTHONPATH="$ROOT" python -c "import duetsim, sys; assert 'paper_2308_01999_b200' in repr(duetsim.statevec), duetsim.__file__"
    PYTHONPATH="$ROOT" python -m pytest -q -p no:cacheprovider "${@:2}" .
    ;;
  *)
    echo "usage: $0 stage|run [pytest args]" >&2
    exit 2
    ;;
esac
