"""Shared test configuration.

Markers: ``gpu`` — needs a CUDA device and the built libdsv.so (run on the
B200 box with ``pytest -m gpu``); everything else runs on CPU.
"""

from __future__ import annotations

import gzip
import os
import pickle
import sys
from functools import lru_cache
from pathlib import Path

for _var in ("OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "OMP_NUM_THREADS"):
    os.environ.setdefault(_var, "1")

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import pytest  # noqa: E402

try:
    from hypothesis import HealthCheck, settings

    settings.register_profile("ci", max_examples=25, deadline=None,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("ci")
except ImportError:  # pragma: no cover
    pass

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU and the built libdsv.so")


@lru_cache(maxsize=None)
def golden(name: str):
    with gzip.open(GOLDEN / f"{name}.pkl.gz", "rb") as fh:
        return pickle.load(fh)["data"]


def gate_from_spec(spec):
    from paper_2308_01999_b200 import gates as G

    if spec["kind"] == "perm":
        return G.PermutationGate(spec["perm"], spec["diag"], spec["targets"], spec["controls"])
    return G.DenseGate(spec["matrix"], spec["targets"], spec["controls"], unitary=spec.get("unitary", True))


def random_state(n: int, rng: np.random.Generator, dtype=np.complex128) -> np.ndarray:
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (v / np.linalg.norm(v)).astype(dtype)


@pytest.fixture(scope="session")
def gpu_available():
    from paper_2308_01999_b200 import _native as N

    if N.device_count() < 1:
        pytest.fail("no CUDA device visible to libdsv (gpu tests must run on the GPU box)")
    return True
