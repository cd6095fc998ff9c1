"""Host-side logic on CPU: gate payload validation, circuit generators and
JSON, fusion (reference semantics, pinned by reference goldens), sharding
plans and transfer accounting.  No GPU, no kernel calls."""

import numpy as np
import pytest

from conftest import gate_from_spec, golden
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import (
    Circuit,
    GateOp,
    gen_qaoa_maxcut,
    gen_qft,
    gen_qv,
    random_gate_sequence,
    to_gates,
)
from paper_2308_01999_b200.core import InvalidArgumentError, bit_permute, bit_permute_array, check_swap_pairs
from paper_2308_01999_b200.fusion import FusionConfig, expand_gate, fuse, fused_matrix
from paper_2308_01999_b200.plan import relabel, relocation_pairs, split_controls, swap_transfer
from oracle import sv_oracle as O


# ---- core / gates ----------------------------------------------------------------

def test_bit_permute_and_pairs():
    assert bit_permute(0b10, [(0, 1)]) == 0b01
    assert bit_permute(12345, []) == 12345
    with pytest.raises(InvalidArgumentError):
        bit_permute(0, [(0, 1), (1, 2)])
    with pytest.raises(InvalidArgumentError):
        check_swap_pairs([(3, 3)])
    with pytest.raises(InvalidArgumentError):
        check_swap_pairs([(0, 64)])
    idx = np.random.default_rng(7).integers(0, 1 << 10, size=200)
    vec = bit_permute_array(idx, [(0, 9), (3, 5)])
    assert all(vec[i] == bit_permute(int(x), [(0, 9), (3, 5)]) for i, x in enumerate(idx))


def test_gate_validation():
    with pytest.raises(InvalidArgumentError):
        G.DenseGate(np.eye(4), (0,))
    with pytest.raises(InvalidArgumentError):
        G.DenseGate(np.eye(2), (0,), controls=((0, 1),))
    with pytest.raises(InvalidArgumentError):
        G.DenseGate(np.ones((2, 2)), (0,))
    G.DenseGate(np.ones((2, 2)), (0,), unitary=False)
    with pytest.raises(InvalidArgumentError):
        G.PermutationGate([0, 0], [1, 1], (0,))
    with pytest.raises(InvalidArgumentError):
        G.PauliString(((0, "Z"), (0, "X")))
    with pytest.raises(InvalidArgumentError):
        G.PauliString(((0, "Q"),))
    assert G.swap(0, 1).to_matrix()[2, 1] == 1
    assert G.cz(0, 1).is_diagonal and not G.x(0).is_diagonal


# ---- circuits ----------------------------------------------------------------------

def test_generator_counts_match_reference():
    c = golden("misc")["counts"]
    assert len(gen_qft(33)) == c["qft33"] == 577
    assert len(gen_qv(33, 30, seed=0)) == c["qv33"] == 480
    assert len(gen_qv(34, 30, seed=0)) == c["qv34"]
    assert len(gen_qft(20)) == c["qft20"] == 220
    for n in (1, 2, 5, 20):
        assert len(gen_qft(n)) == n + n * (n - 1) // 2 + n // 2
    assert [tuple(op.targets) for op in gen_qv(6, 5, seed=3).ops] == [tuple(t) for t in golden("misc")["qv6_targets"]]


def test_qaoa_and_json_roundtrip(tmp_path):
    c = gen_qaoa_maxcut([(0, 1), (1, 2), (2, 0)], p=2, seed=1)
    assert c.num_qubits == 3 and len(c) == 3 + 2 * 6
    with pytest.raises(InvalidArgumentError):
        gen_qaoa_maxcut([], p=1)
    rng = np.random.default_rng(0)
    ops = [GateOp("h", (), (0,)), GateOp("rz", (0.3,), (1,)), GateOp("x", (), (0,), ((1, 1),)),
           GateOp("unitary", (), (0, 2), (), G.random_unitary(4, rng))]
    circ = Circuit(3, ops)
    path = tmp_path / "c.json"
    circ.save(path)
    back = Circuit.load(path)
    a = O.run_circuit(to_gates(circ), 3)
    b = O.run_circuit(to_gates(back), 3)
    np.testing.assert_allclose(a, b, atol=1e-15)
    with pytest.raises(InvalidArgumentError):
        Circuit(2, [GateOp("h", (), (5,))])


def test_random_gate_sequence_reproduces_reference_oracle():
    for case in golden("misc")["random_gate_sequence"]:
        seq = random_gate_sequence(case["n"], case["count"], np.random.default_rng(case["seed"]),
                                   max_arity=case["max_arity"])
        ref = [gate_from_spec(s) for s in case["gates"]]
        assert len(seq) == len(ref)
        for a, b in zip(seq, ref):
            assert type(a) is type(b) and a.targets == b.targets
            if isinstance(a, G.PermutationGate):
                np.testing.assert_array_equal(a.permutation, b.permutation)
                np.testing.assert_array_equal(a.diagonal, b.diagonal)
            else:
                np.testing.assert_array_equal(a.matrix, b.matrix)


# ---- fusion --------------------------------------------------------------------------

def test_fusion_matches_reference_goldens():
    fam = golden("fusion")
    for case in fam["cases"]:
        gates = [gate_from_spec(s) for s in case["gates"]]
        fc = fuse(gates, FusionConfig(*case["cfg"]))
        assert fc.provenance == case["provenance"], (case["name"], case["cfg"])
        assert len(fc.gates) == len(case["fused"])
        for fg, spec, passthrough in zip(fc.gates, case["fused"], case["passthrough"]):
            assert any(fg is g for g in gates) == passthrough
            ref = gate_from_spec(spec)
            assert type(fg) is type(ref) and tuple(fg.targets) == tuple(ref.targets)
            if isinstance(fg, G.PermutationGate):
                np.testing.assert_array_equal(fg.permutation, ref.permutation)
                np.testing.assert_array_equal(fg.diagonal, ref.diagonal)  # same op order => bit-equal
            else:
                np.testing.assert_allclose(fg.matrix, ref.matrix, atol=1e-13)
        out = O.run_circuit(fc.gates, case["n"])
        np.testing.assert_allclose(out, case["out"], atol=1e-10)


def test_fusion_counts_at_benchmark_scale():
    counts = golden("fusion")["counts"]
    assert len(fuse(to_gates(gen_qft(33)), FusionConfig(5, 6))) == counts["qft33_5_6"] == 152
    assert len(fuse(to_gates(gen_qft(33)), FusionConfig(5, 10))) == counts["qft33_5_10"]
    assert len(fuse(to_gates(gen_qv(34, 30, seed=0)), FusionConfig(4, 6))) == counts["qv34_4_6"]
    assert len(fuse(to_gates(gen_qft(20)), FusionConfig(5, 6))) == counts["qft20_5_6"]


def test_fusion_unit_behaviour():
    fc = fuse([G.h(0), G.h(0)], FusionConfig(max_fused_gate_size=2))
    assert len(fc) == 1
    np.testing.assert_allclose(fc.gates[0].matrix, np.eye(2), atol=1e-15)
    rng = np.random.default_rng(1)
    big = G.unitary(G.random_unitary(32, rng), (0, 1, 2, 3, 4))
    fc = fuse([big, G.h(0)], FusionConfig(max_fused_gate_size=2))
    assert len(fc) == 2 and fc.gates[0] is big
    g = fused_matrix([G.cx(0, 1), G.cx(0, 1)], [0, 1])
    np.testing.assert_allclose(g.matrix, np.eye(4), atol=1e-15)
    np.testing.assert_allclose(expand_gate(G.x(0), [0, 1]), O.full_operator(2, G.PAULI_MATS["X"], (0,)))
    with pytest.raises(InvalidArgumentError):
        fused_matrix([G.x(5)], [0, 1])
    with pytest.raises(InvalidArgumentError):
        FusionConfig(0, 3)
    n, dmax = 8, 4
    circ = [G.rz(0.1 * (q + 1), q) for q in range(n)] + [G.cz(q, q + 1) for q in range(0, n - 1, 2)]
    fc = fuse(circ, FusionConfig(2, dmax))
    assert all(isinstance(x, G.PermutationGate) and x.is_diagonal for x in fc.gates)
    assert len(fc) == -(-n // dmax)


def test_fusion_idempotent_on_random_circuits():
    for seed in range(10):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 8))
        seq = random_gate_sequence(n, int(rng.integers(3, 50)), rng, max_arity=3)
        cfg = FusionConfig(4, 5)
        once = fuse(seq, cfg)
        assert len(fuse(once.gates, cfg)) == len(once)


# ---- sharding plans ----------------------------------------------------------------------

def _replay_stats(n, g, workers, gates):
    """Host replay of SegmentedStateVector.run's planning (no data)."""
    nloc = n - g
    qmap = list(range(n))
    stats = dict(num_reorders=0, num_messages=0, amplitudes_moved=0,
                 amplitudes_moved_intra_worker=0, amplitudes_moved_inter_worker=0)
    for i, gate in enumerate(gates):
        pairs = relocation_pairs(qmap, nloc, [qmap[q] for q in gate.targets], gates[i + 1:])
        if pairs:
            ex, moved, intra, inter = swap_transfer(pairs, nloc, g, workers)
            if ex:
                stats["num_reorders"] += 1
                stats["num_messages"] += 2 * ex
                stats["amplitudes_moved"] += moved
                stats["amplitudes_moved_intra_worker"] += intra
                stats["amplitudes_moved_inter_worker"] += inter
            qmap = relabel(qmap, pairs)
        split_controls(qmap, nloc, gate.controls)
    return stats, qmap


def test_distributed_plan_matches_reference_runs():
    for case in golden("distsim")["runs"]:
        gates = [gate_from_spec(s) for s in case["gates"]]
        stats, qmap = _replay_stats(case["n"], case["g"], case["workers"], gates)
        assert stats == case["stats"]
        assert qmap == case["qubit_map"]


def test_swap_transfer_matches_reference_swaps():
    for c in golden("distsim")["swaps"]:
        ex, moved, intra, inter = swap_transfer(c["pairs"], c["n"] - c["g"], c["g"], c["workers"])
        st = c["stats"]
        assert st["num_reorders"] == (1 if ex else 0)
        assert st["num_messages"] == 2 * ex
        assert st["amplitudes_moved"] == moved
        assert st["amplitudes_moved_intra_worker"] == intra
        assert st["amplitudes_moved_inter_worker"] == inter
        assert relabel(list(range(c["n"])), c["pairs"]) == c["qubit_map"]


def test_relocation_prefers_idle_victims_and_rejects_overflow():
    # q3 global (n=4, g=1); upcoming uses q0, q1 as targets -> victim is bit 2
    gates = [G.h(0), G.h(1), G.h(3)]
    assert relocation_pairs([0, 1, 2, 3], 3, [3], gates) == [(3, 2)]
    assert relocation_pairs([0, 1, 2, 3], 3, [3], []) == [(3, 0)]
    with pytest.raises(InvalidArgumentError):
        relocation_pairs([0, 1, 2, 3], 2, [0, 2, 3], [])


def test_fold_ops_stream_matches_fuse_fold():
    """fold_ops (the generator the e2e path streams into run_circuit_sv)
    yields exactly fuse_fold's ops, window by window."""
    from paper_2308_01999_b200.circuits import gen_qft, gen_qv, to_gates
    from paper_2308_01999_b200.fusion_fold import fold_ops, fuse_fold

    for gates, k in ((to_gates(gen_qft(17)), 5), (to_gates(gen_qv(9, depth=6, seed=2)), 4)):
        a = fuse_fold(gates, k).ops
        b = list(fold_ops(gates, k))
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert type(x) is type(y)
            if hasattr(x, "matrix"):
                assert x.targets == y.targets
                np.testing.assert_array_equal(x.matrix, y.matrix)
