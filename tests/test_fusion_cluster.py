"""Cluster-merging fuser (paper_2308_01999_b200/fusion_cluster.py): the fused
circuit equals the original on the CPU oracle for every window size,
layered circuits fuse into fewer windows than the reference / fold fusers,
and fuse_auto keeps the fold fuser's phase folding where it wins (QFT)."""

import numpy as np
import pytest

from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qaoa_maxcut, gen_qft, gen_qv, random_gate_sequence, to_gates
from paper_2308_01999_b200.fusion import FusionConfig, fuse
from paper_2308_01999_b200.fusion_cluster import fuse_auto, fuse_cluster
from paper_2308_01999_b200.fusion_fold import fuse_fold


def _circuits():
    rng = np.random.default_rng(3)
    ctrl = [G.x(2, controls=((0, 1),)), G.DenseGate(G.random_unitary(4, rng), (1, 3), controls=((5, 0),)),
            G.unitary(G.random_unitary(8, rng), (4, 0, 6))]
    return [
        ("qv8", 8, to_gates(gen_qv(8, 12, seed=1))),
        ("random7", 7, random_gate_sequence(7, 80, rng, max_arity=3) + ctrl),
        ("qft9", 9, to_gates(gen_qft(9))),
        ("qaoa8", 8, to_gates(gen_qaoa_maxcut([(q, (q + 1) % 8) for q in range(8)], p=2, seed=4))),
    ]


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("name,n,circ", _circuits())
def test_cluster_fusion_equals_circuit(name, n, circ, k):
    want = O.run_circuit(circ, n)
    fc = fuse_cluster(circ, k)
    assert sorted(i for p in fc.provenance for i in p) == list(range(len(circ)))
    for op in fc.ops:
        assert len(op.qubits) <= max(k, max(len(g.qubits) for g in circ))
    assert np.abs(O.run_circuit(fc.ops, n) - want).max() < 1e-12


def test_layered_circuits_fuse_into_fewer_windows():
    for n, k, want in ((33, 5, 130), (34, 4, 181), (33, 4, 169), (33, 6, 99)):
        g = to_gates(gen_qv(n, 30, seed=0))
        got = fuse_cluster(g, k).data_passes
        assert got == want
        assert got < len(fuse(g, FusionConfig(k, 6)).gates)
        assert got < fuse_fold(g, k).data_passes


def test_auto_keeps_phase_folding_for_qft():
    g = to_gates(gen_qft(33))
    assert fuse_auto(g, 5).data_passes == fuse_fold(g, 5).data_passes == 7
    q = to_gates(gen_qv(33, 30, seed=0))
    assert fuse_auto(q, 5).data_passes == 130


def test_oversized_gates_pass_through():
    rng = np.random.default_rng(9)
    n = 6
    circ = [G.h(0), G.unitary(G.random_unitary(16, rng), (0, 1, 2, 3)), G.cx(3, 4), G.h(5)]
    fc = fuse_cluster(circ, 2)
    assert any(op is circ[1] for op in fc.ops)
    assert np.abs(O.run_circuit(fc.ops, n) - O.run_circuit(circ, n)).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_cluster_fused_qv_on_gpu(dtype, gpu_available):
    """Cluster-fused quantum volume (k = 4 and 5 dense windows: tensor-core
    and CUDA-core kernels) on the B200 against the oracle."""
    from conftest import assert_state_close
    from paper_2308_01999_b200.statevec import StateVector

    n = 18
    circ = to_gates(gen_qv(n, 10, seed=5))
    want = O.run_circuit(circ, n)
    for k in (4, 5):
        sv = StateVector(n, dtype=dtype)
        for op in fuse_cluster(circ, k).ops:
            sv.apply(op)
        assert_state_close(sv.logical_amplitudes(), want, dtype)
