"""CUDA-graph capture and replay of gate sequences (StateVector.capture,
include/dsv.h dsv_capture_* / dsv_graph_*): every gate family — kernel-
parameter matrices, per-gate device tables (diagonals, generic k >= 7,
tensor-core digits and phase tables), relabelling swaps of the fold fuser —
replays to the oracle's state, repeatedly, and host round trips are refused
while recording."""

import numpy as np
import pytest

from conftest import assert_state_close, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, random_gate_sequence, to_gates
from paper_2308_01999_b200.core import InvalidArgumentError
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_capture_and_replay_random_circuit(dtype):
    n = 14
    rng = np.random.default_rng(21)
    gates = random_gate_sequence(n, 60, rng, max_arity=3)
    gates += [G.DenseGate(G.random_unitary(128, rng), tuple(range(2, 9))),                # generic k = 7
              G.DenseGate(G.random_unitary(32, rng), (3, 5, 7, 9, 11)),                   # tensor cores (c64)
              G.PermutationGate(rng.permutation(8), np.exp(1j * rng.uniform(0, 6, 8)), (0, 4, 13), ((6, 1),))]
    st = random_state(n, rng, dtype)
    sv = StateVector.from_amplitudes(st)
    with sv.capture() as rec:
        for g in gates:
            sv.apply(g)
    want = O.run_circuit(gates, n, state=st.astype(np.complex128))
    assert_state_close(sv.amplitudes, want, dtype)
    for _ in range(2):  # replay from the same input, twice
        sv.amplitudes = st
        rec.replay()
        assert_state_close(sv.amplitudes, want, dtype)
    rec.close()


def test_capture_fold_fused_qft_with_relabels():
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 16
    sv = StateVector(n, dtype=np.complex64)
    ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
    with sv.capture() as rec:
        for op in ops:
            sv.apply(op)
    want = O.run_circuit(to_gates(gen_qft(n)), n)
    assert_state_close(sv.logical_amplitudes(), want, np.complex64)
    sv.native.set_basis(0)
    sv.bit_map = list(rec.start_map)
    rec.replay()
    assert sv.bit_map == rec.end_map
    assert_state_close(sv.logical_amplitudes(), want, np.complex64)
    sv.bit_map = [1, 0] + list(range(2, n))
    with pytest.raises(InvalidArgumentError):
        rec.replay()


def test_host_round_trips_refused_while_capturing():
    sv = StateVector(8, dtype=np.complex128)
    with pytest.raises(InvalidArgumentError):
        with sv.capture():
            sv.apply(G.h(0))
            sv.probabilities([0])
    # the state is still usable afterwards
    sv.apply(G.h(1))
    assert abs(sv.norm_squared() - 1.0) < 1e-12
