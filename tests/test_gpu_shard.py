"""The single-process sharded engine (shard.py) on a B200: P = 2/4/8 segments
driven from one host thread through libdsv.  On a 1-GPU box every segment
sits on cuda:0 (the driver's round-end GPU is a single B200); the kernels,
the masked exchange (both halves, two streams, event joins) and the group
reductions are the ones an 8-GPU run uses, only the peer pointers are local.

Parity bars (BASELINE.json north_star): bit-exact for permutations,
diagonals and index-bit swaps; max |d| <= 1e-5 (c64) / 1e-12 (c128) and
fidelity >= 1 - 1e-6 for dense gates, against the CPU oracle and across P
(P-invariance, SURVEY.md §7.3 hard part 4: the only full-size parity route
for BASELINE configs 4 and 5).
"""

import numpy as np
import pytest

from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, gen_qv, random_gate_sequence, to_gates
from paper_2308_01999_b200.core import bit_permute_array
from paper_2308_01999_b200.shard import ShardedStateVector
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu

TOL = {np.complex64: 1e-5, np.complex128: 1e-12}


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


def _fidelity(a, b):
    return abs(np.vdot(a.astype(np.complex128), b.astype(np.complex128))) ** 2 / (
        np.vdot(a, a).real * np.vdot(b, b).real)


def _run(n, P, gates, dtype):
    sv = ShardedStateVector(n, [0] * P, dtype)
    sv.run(gates)
    out = sv.gather_logical()
    stats = sv.stats.as_dict()
    sv.close()
    return out, stats


def _perm_diag_circuit(n, count, rng, max_arity=3):
    """random_gate_sequence restricted to its diagonal / permutation kinds."""
    out = []
    while len(out) < count:
        g = random_gate_sequence(n, 1, rng, max_arity)[0]
        if isinstance(g, G.PermutationGate):
            out.append(g)
    return out


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_permutation_circuit_bit_identical_across_P(dtype):
    """Generalised permutations / diagonals (NumPy FMA-form product) and the
    exchanges are bit-exact: P = 1, 2, 4, 8 give IEEE-identical states, equal
    to the CPU oracle's."""
    n = 20
    rng = np.random.default_rng(3)
    gates = _perm_diag_circuit(n, 120, rng)
    gates += [G.x(19, controls=((18, 1),)), G.PermutationGate([1, 0], [1j, -1], (19,), ((0, 0),))]
    want = O.run_circuit(gates, n, dtype=dtype)
    outs = [_run(n, P, gates, dtype)[0] for P in (1, 2, 4, 8)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert np.array_equal(outs[0], want)


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_random_circuit_vs_oracle_across_P(dtype):
    """Config 5's generator (random 1-/2-qubit dense, diagonal, permutation
    gates) at n = 20 on 2 / 4 / 8 segments against the CPU oracle."""
    n = 20
    gates = random_gate_sequence(n, 200, np.random.default_rng(0), max_arity=2)
    want = O.run_circuit(gates, n)
    for P in (2, 4, 8):
        got, stats = _run(n, P, gates, dtype)
        assert np.abs(got - want).max() <= TOL[dtype], P
        assert _fidelity(got, want) >= 1 - 1e-6
        assert stats["num_reorders"] > 0


def test_qv_c128_two_vs_four_segments():
    """Config 4's generator (quantum volume, c128) at n = 16: 2 and 4
    segments agree within 1e-12 of each other and of the oracle."""
    n = 16
    gates = to_gates(gen_qv(n, 12, seed=0))
    want = O.run_circuit(gates, n)
    s2, _ = _run(n, 2, gates, np.complex128)
    s4, _ = _run(n, 4, gates, np.complex128)
    assert np.abs(s2 - s4).max() <= 1e-12
    assert np.abs(s2 - want).max() <= 1e-12
    assert _fidelity(s4, want) >= 1 - 1e-12


def test_expectation_and_marginals_vs_oracle():
    """Config 5's observables: <Z0 X17 Y19> and sum_q <Z_q> on a sharded
    random c64 state (n = 20, P = 8) vs the oracle."""
    n = 20
    gates = random_gate_sequence(n, 120, np.random.default_rng(7), max_arity=2)
    want = O.run_circuit(gates, n)
    sv = ShardedStateVector(n, [0] * 8, np.complex64)
    sv.run(gates)
    p = G.PauliString(((0, "Z"), (17, "X"), (19, "Y")))
    ev = sv.expectation([p])
    ev_want = O.expectation_pauli(want, n, p.factors, p.coefficient)
    assert abs(ev - ev_want) <= 1e-5
    zs = sv.expectation([G.PauliString(((q, "Z"),)) for q in range(n)])
    zs_want = sum(O.expectation_pauli(want, n, ((q, "Z"),), 1.0) for q in range(n))
    assert abs(zs - zs_want) <= 1e-4
    pr = sv.probabilities([19, 0, 7])
    assert np.abs(pr - O.marginal(want, n, [19, 0, 7])).max() <= 1e-6
    assert abs(sv.norm_squared() - 1.0) <= 1e-5
    # the relocation for X on a global qubit left the logical state intact
    assert np.abs(sv.gather_logical() - want).max() <= 1e-5
    sv.close()


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("P,pairs", [
    (2, [(19, 0)]), (2, [(19, 1)]), (4, [(19, 0), (18, 5)]), (8, [(17, 0), (18, 1), (19, 2)]),
    (8, [(19, 12), (18, 13)]), (8, [(19, 18), (0, 3)]), (4, [(19, 17), (18, 0)]),
])
def test_distributed_swap_bit_exact(dtype, P, pairs):
    """Batched masked exchanges (incl. the 16-byte lane mode for amplitude
    bit 0 in complex64) equal the full-vector bit permutation exactly."""
    n = 20
    rng = np.random.default_rng(2)
    full = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(dtype)
    sv = ShardedStateVector(n, [0] * P, dtype)
    nloc = sv.local_bits
    for s, seg in enumerate(sv.segs):
        seg.upload(np.ascontiguousarray(full[s << nloc:(s + 1) << nloc]))
    sv.distributed_index_bit_swap(pairs)
    got = np.concatenate(sv.physical_segments())
    want = np.empty_like(full)
    want[bit_permute_array(np.arange(full.size), pairs)] = full
    assert np.array_equal(got, want)
    sv.close()


def test_fold_fused_qft_sharded():
    """The headline workload's fold-fused QFT from |x> on 8 segments (n = 22):
    the DFT column, one global<->local reorder."""
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n, x = 22, 987654
    ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
    sv = ShardedStateVector(n, [0] * 8, np.complex64)
    # |x> written through the segment holding it (identity map before run)
    sv.reset()
    sv.segs[0].set_zero()
    sv.segs[x >> sv.local_bits].set_basis(x & ((1 << sv.local_bits) - 1))
    sv._basis0 = False
    sv.run(ops)
    y = np.arange(1 << n)
    dft = np.exp(2j * np.pi * x * y / (1 << n)) / np.sqrt(1 << n)
    got = sv.gather_logical()
    assert np.abs(got - dft).max() <= 1e-5
    assert _fidelity(got, dft) >= 1 - 1e-6
    sv.close()
    # from |0>: the initial placement leaves one reorder
    sv = ShardedStateVector(n, [0] * 8, np.complex64)
    sv.run(ops)
    assert sv.stats.num_reorders == 1
    assert np.abs(sv.gather_logical() - 2 ** (-n / 2)).max() <= 1e-6
    sv.close()


def test_sharded_equals_single_segment_statevector():
    """P = 4 vs the single-segment StateVector on a mixed c64 circuit."""
    n = 21
    gates = to_gates(gen_qft(n)) + random_gate_sequence(n, 60, np.random.default_rng(9), max_arity=3)
    single = StateVector(n, dtype=np.complex64)
    for g in gates:
        single.apply(g)
    got, _ = _run(n, 4, gates, np.complex64)
    assert np.abs(got - single.logical_amplitudes()).max() <= 1e-5


@pytest.mark.parametrize("P", [2, 4])
def test_fold_and_cluster_fused_c128_sharded(P):
    """complex128 sharded runs of both opt-in fusers' ops (phased windows with
    global outside qubits folded per segment; cluster-fused dense windows)."""
    from paper_2308_01999_b200.fusion_cluster import fuse_cluster
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 16
    for ops, want in ((fuse_fold(to_gates(gen_qft(n)), 5).ops, O.run_circuit(to_gates(gen_qft(n)), n)),
                      (fuse_cluster(to_gates(gen_qv(n, 8, seed=3)), 4).ops,
                       O.run_circuit(to_gates(gen_qv(n, 8, seed=3)), n))):
        sv = ShardedStateVector(n, [0] * P, np.complex128)
        sv.run(ops)
        assert np.abs(sv.gather_logical() - want).max() <= 1e-12
        sv.close()
