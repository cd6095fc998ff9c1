"""Streamed dump / load: chunked GPU gathers in logical
order, byte-identical to the reference file format (statevec.py:332-351)."""

import struct

import numpy as np
import pytest

from conftest import random_state
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_streamed_dump_load_round_trip(tmp_path, monkeypatch, dtype):
    monkeypatch.setattr(StateVector, "DUMP_CHUNK", 1 << 10)  # many chunks
    rng = np.random.default_rng(3)
    n = 14
    st = random_state(n, rng, dtype)
    sv = StateVector.from_amplitudes(st)
    sv.swap_index_bits([(0, 9), (3, 12)])  # physical order != logical order
    path = tmp_path / "s.bin"
    sv.dump(path)
    raw = path.read_bytes()
    assert struct.unpack("<Q", raw[:8])[0] == n and len(raw) == 8 + (16 << n)
    np.testing.assert_array_equal(np.frombuffer(raw[8:], "<f8").view(np.complex128), st.astype(np.complex128))
    back = StateVector.load(path)
    np.testing.assert_array_equal(back.logical_amplitudes(), st.astype(np.complex128))
    narrow = StateVector.load(path, dtype=np.complex64)
    np.testing.assert_array_equal(narrow.logical_amplitudes(), st.astype(np.complex64))
