"""The reference's OWN hot-path tests (pkg/tests/test_core.py,
test_statevec.py, test_fusion.py, test_distsim.py + its oracles.py /
conftest.py), unmodified, against the drop-in `duetsim` package on the GPU.

The files are staged by `tools/ref_suite.sh stage` in the build container
(the only place /root/reference exists) into the git-ignored ref_suite/,
which travels to the GPU box with the repository snapshot; no reference
source is committed.  Without the staged copy the test is skipped."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SUITE = ROOT / "ref_suite"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (SUITE / "SHA256SUMS").exists(), reason="reference suite not staged (tools/ref_suite.sh stage)")
def test_reference_hot_path_suite_passes_against_the_drop_in(gpu_available):
    res = subprocess.run(["bash", str(ROOT / "tools" / "ref_suite.sh"), "run"], capture_output=True, text=True,
                         timeout=900)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
