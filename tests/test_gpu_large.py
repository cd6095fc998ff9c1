"""GPU parity at sizes where the CPU oracle is slow or infeasible, through
size-independent properties (SURVEY.md §7.3 hard part 4):

* bit-exact involutions / inverses for permutations and swaps at n = 28;
* U then U^dagger round trips (tolerance) and norm preservation;
* analytic QFT|0> = uniform 2^(-n/2);
* P-invariance: segmented runs equal the single-segment run;
* oracle parity at n = 22-24 where numpy still finishes in seconds.
"""

import numpy as np
import pytest

from conftest import assert_state_close, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, random_gate_sequence, to_gates
from paper_2308_01999_b200.distsim import SegmentedStateVector
from paper_2308_01999_b200.fusion import FusionConfig, fuse
from paper_2308_01999_b200.statevec import StateVector, run_circuit_sv

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


def _dagger(g):
    if isinstance(g, G.PermutationGate):
        inv = np.empty_like(g.permutation)
        inv[g.permutation] = np.arange(g.permutation.size)
        return G.PermutationGate(inv, np.conj(g.diagonal)[inv], g.targets, g.controls)
    return G.DenseGate(g.matrix.conj().T, g.targets, g.controls)


def test_large_swap_and_permutation_involutions_bit_exact():
    n = 28
    rng = np.random.default_rng(0)
    sv = StateVector(n, dtype=np.complex64)
    for q in range(0, n, 3):
        sv.apply(G.ry(0.1 + q, q))
    sv.apply(G.unitary(G.random_unitary(8, rng), (0, 13, 27)))
    before = sv.native.download()
    for pairs in ([(0, 27)], [(1, 2), (5, 26), (3, 14)], [(0, 1)]):
        sv.swap_index_bits(pairs)
        sv.swap_index_bits(pairs)
        np.testing.assert_array_equal(sv.native.download(), before)
    for targets in ((0,), (1, 20), (27, 3, 9)):
        k = len(targets)
        perm = rng.permutation(1 << k)
        g = G.PermutationGate(perm, np.ones(1 << k), targets, ((5, 1),) if k < 3 else ())
        sv.apply(g)
        sv.apply(_dagger(g))
        np.testing.assert_array_equal(sv.native.download(), before)


@pytest.mark.parametrize("dtype,n", [(np.complex64, 28), (np.complex128, 27)])
def test_large_round_trip_and_norm(dtype, n):
    rng = np.random.default_rng(1)
    gates = random_gate_sequence(n, 40, rng, max_arity=3)
    gates += [G.DenseGate(G.random_unitary(1 << k, rng), tuple(rng.permutation(n)[:k].tolist()))
              for k in (4, 5)]
    sv = StateVector(n, dtype=dtype)
    sv.apply(G.h(0))
    start = sv.native.download()
    for g in gates:
        sv.apply(g)
    assert abs(sv.norm_squared() - 1.0) < (1e-5 if dtype == np.complex64 else 1e-12)
    for g in reversed(gates):
        sv.apply(_dagger(g))
    assert_state_close(sv.native.download(), start, dtype)


def test_qft_uniform_at_26_qubits_fused():
    n = 26
    fc = fuse(to_gates(gen_qft(n)), FusionConfig(5, 6))
    sv = run_circuit_sv(fc.gates, n, dtype=np.complex64)
    a = sv.native.download()
    assert np.abs(a - 2.0 ** (-n / 2)).max() < 1e-6


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_oracle_parity_at_22_qubits(dtype):
    n = 22
    rng = np.random.default_rng(2)
    st = random_state(n, rng, dtype)
    gates = random_gate_sequence(n, 12, rng, max_arity=3)
    gates.append(G.PermutationGate(np.arange(64), np.exp(1j * rng.uniform(0, 6, 64)), tuple(range(16, 22))))
    want = O.run_circuit(gates, n, dtype=dtype, state=st)
    sv = StateVector.from_amplitudes(st)
    for g in gates:
        sv.apply(g)
    assert_state_close(sv.native.download(), want, dtype)


def test_diagonal_bit_exact_at_24_qubits():
    n = 24
    rng = np.random.default_rng(3)
    st = random_state(n, rng, np.complex64)
    sv = StateVector.from_amplitudes(st)
    want = st.copy()
    for targets, ctrl in (((0, 1, 2, 3, 4, 5), ()), ((18, 23), ((2, 1),)), ((7,), ((0, 1), (20, 0)))):
        d = np.exp(1j * rng.uniform(0, 6.3, 1 << len(targets)))
        g = G.PermutationGate(np.arange(d.size), d, targets, ctrl)
        sv.apply(g)
        O.apply_genperm(want, n, g.permutation, g.diagonal, list(targets), list(ctrl))
    np.testing.assert_array_equal(sv.native.download(), want)


@pytest.mark.parametrize("gbits", [1, 2, 3])
def test_segmented_equals_single_segment(gbits):
    n = 20
    gates = to_gates(gen_qft(n)) + random_gate_sequence(n, 30, np.random.default_rng(gbits), max_arity=2)
    ref = run_circuit_sv(gates, n).amplitudes
    with SegmentedStateVector(n, gbits, workers=2) as ssv:
        ssv.run(gates)
        got = ssv.to_statevector().amplitudes
        assert ssv.stats.num_reorders > 0
    assert_state_close(got, ref, np.complex128)


def test_segmented_fold_ops_match_single():
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 16
    gates = to_gates(gen_qft(n)) + random_gate_sequence(n, 20, np.random.default_rng(9), max_arity=2)
    ref = run_circuit_sv(gates, n).amplitudes
    fc = fuse_fold(gates, 4)
    with SegmentedStateVector(n, 3) as ssv:
        ssv.run(fc.ops)
        np.testing.assert_allclose(ssv.to_statevector().amplitudes, ref, atol=1e-12)


def test_segmented_expectation_matches_single():
    n = 16
    rng = np.random.default_rng(8)
    gates = random_gate_sequence(n, 30, rng, max_arity=2)
    ref = run_circuit_sv(gates, n)
    obs = [G.PauliString(((0, "Z"), (7, "X"), (15, "Y")), 0.5), G.PauliString(((14, "Z"), (15, "Z")))]
    with SegmentedStateVector(n, 2) as ssv:
        ssv.run(gates)
        got = ssv.expectation(obs)
        assert abs(ssv.norm_squared() - 1.0) < 1e-10
        np.testing.assert_allclose(ssv.to_statevector().amplitudes, ref.amplitudes, atol=1e-12)
    assert abs(got - ref.expectation(obs)) < 1e-10


def _sample_chunks(nat, nbits, nchunks=8, chunk=1 << 17):
    begins = np.linspace(0, (1 << nbits) - chunk, nchunks).astype(np.int64)
    return np.concatenate([nat.download(np.empty(chunk, nat.dtype), int(b), chunk) for b in begins])


def test_headline_size_n33_c64_properties():
    """At the headline size (n = 33 complex64, 64 GiB): a generalised
    permutation followed by its inverse, an index-bit swap applied twice and
    a k = 5 tensor-core window followed by its adjoint leave the state
    unchanged — bit-exactly for the permutation and swap (compared on 1 M
    sampled amplitudes) and within the c64 bars for the window."""
    n = 33
    rng = np.random.default_rng(33)
    sv = StateVector(n, dtype=np.complex64)
    for q in (0, 7, 16, 25, 32):
        sv.apply(G.ry(0.3 + q, q))
    sv.apply(G.unitary(G.random_unitary(4, rng), (1, 30)))
    nat = sv.native
    before = _sample_chunks(nat, n)
    perm = G.PermutationGate(rng.permutation(8), np.ones(8), (2, 19, 31), ((5, 1),))
    sv.apply(perm)
    sv.apply(_dagger(perm))
    np.testing.assert_array_equal(_sample_chunks(nat, n), before)
    sv.swap_index_bits([(0, 32), (3, 17)])
    sv.swap_index_bits([(0, 32), (3, 17)])
    np.testing.assert_array_equal(_sample_chunks(nat, n), before)
    w = G.DenseGate(G.random_unitary(32, rng), (4, 9, 14, 21, 27))
    sv.apply(w)
    sv.apply(_dagger(w))
    assert_state_close(_sample_chunks(nat, n), before, np.complex64)
    assert abs(sv.norm_squared() - 1.0) < 1e-5
