"""The opt-in phase-folding fuser (fusion_fold.py): exact equivalence with the
unfused circuit (CPU, oracle as checker) and the GPU phased-window kernel
against the same oracle."""

import numpy as np
import pytest

from conftest import assert_state_close, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qaoa_maxcut, gen_qft, gen_qv, random_gate_sequence, to_gates
from paper_2308_01999_b200.fusion_fold import PhasedDenseGate, QubitSwap, fuse_fold


def run_folded_oracle(fc, n, state=None):
    """Apply fold-fuser ops on the host with the oracle; returns logical amps."""
    amps = np.zeros(1 << n, complex) if state is None else state.astype(complex).copy()
    if state is None:
        amps[0] = 1
    bm = list(range(n))
    idx = np.arange(1 << n)
    for op in fc.ops:
        if isinstance(op, QubitSwap):
            bm[op.a], bm[op.b] = bm[op.b], bm[op.a]
        elif isinstance(op, PhasedDenseGate):
            ph = np.zeros(1 << n)
            for a, b, t in op.cross:
                ph += t * (((idx >> bm[a]) & 1) & ((idx >> bm[b]) & 1))
            for b, t in op.outside:
                ph += t * ((idx >> bm[b]) & 1)
            amps *= np.exp(1j * ph)
            O.apply_dense(amps, n, op.matrix, [bm[q] for q in op.targets])
        else:
            O.apply_gate(amps, n, op, bm)
    return O.access(amps, n, bm)


def controlled_mix(n, count, rng):
    seq = []
    for _ in range(count):
        kind = rng.integers(0, 6)
        a, b, c = (int(x) for x in rng.choice(n, size=3, replace=False))
        if kind == 0:
            seq.append(G.cp(float(rng.uniform(0, 6.3)), a, b))
        elif kind == 1:
            seq.append(G.rzz(float(rng.uniform(0, 6.3)), a, b))
        elif kind == 2:
            seq.append(G.h(a))
        elif kind == 3:
            seq.append(G.x(a, controls=((b, int(rng.integers(0, 2))),)))
        elif kind == 4:
            seq.append(G.p(float(rng.uniform(0, 6.3)), a, controls=((b, 0),)))
        else:
            seq.append(G.swap(a, c) if rng.random() < 0.5 else G.rz(0.7, a))
    return seq


CIRCUITS = [
    ("qft9", 9, lambda: to_gates(gen_qft(9))),
    ("qv8", 8, lambda: to_gates(gen_qv(8, 6, 2))),
    ("qaoa8", 8, lambda: to_gates(gen_qaoa_maxcut([(i, (i + 1) % 8) for i in range(8)] + [(0, 4), (1, 6)], p=2))),
    ("random", 7, lambda: random_gate_sequence(7, 60, np.random.default_rng(3), 3)),
    ("mix", 7, lambda: controlled_mix(7, 80, np.random.default_rng(4))),
]


@pytest.mark.parametrize("name,n,make", CIRCUITS)
@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_fold_fuser_equivalent_to_unfused(name, n, make, k):
    gates = make()
    fc = fuse_fold(gates, k)
    covered = sorted(i for grp in fc.provenance for i in grp)
    assert covered == list(range(len(gates)))
    for op in fc.ops:
        if isinstance(op, PhasedDenseGate):
            assert len(op.targets) <= k
            assert not set(b for _, b, _ in op.cross) & set(op.targets)
    np.testing.assert_allclose(run_folded_oracle(fc, n), O.run_circuit(gates, n), atol=1e-12)


def test_fold_fuser_pass_counts():
    fc = fuse_fold(to_gates(gen_qft(33)), 5)
    assert fc.data_passes == 7                     # vs 152 reference windows
    assert sum(isinstance(o, QubitSwap) for o in fc.ops) == 16
    fc4 = fuse_fold(to_gates(gen_qft(33)), 4)
    assert fc4.data_passes == 9


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("name,n,make", CIRCUITS)
def test_fold_ops_on_gpu_match_oracle(dtype, name, n, make, gpu_available):
    from paper_2308_01999_b200.statevec import StateVector

    gates = make()
    rng = np.random.default_rng(7)
    st = random_state(n, rng, dtype)
    want = O.run_circuit(gates, n, dtype=np.complex128, state=st)
    for k in (3, 5):
        fc = fuse_fold(gates, k)
        sv = StateVector.from_amplitudes(st)
        for op in fc.ops:
            sv.apply(op)
        assert_state_close(sv.logical_amplitudes(), want, dtype)


@pytest.mark.gpu
def test_fold_qft_large_uniform(gpu_available):
    from paper_2308_01999_b200.statevec import StateVector

    n = 26
    sv = StateVector(n, dtype=np.complex64)
    for op in fuse_fold(to_gates(gen_qft(n)), 5).ops:
        sv.apply(op)
    a = sv.native.download()
    assert np.abs(a - 2.0 ** (-n / 2)).max() < 1e-6
    # QFT|x> = DFT column: start from a basis state at n = 14 (phases exercised)
    n = 14
    x = 12345
    st = np.zeros(1 << n, np.complex64)
    st[x] = 1
    sv = StateVector.from_amplitudes(st)
    for op in fuse_fold(to_gates(gen_qft(n)), 5).ops:
        sv.apply(op)
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * x * y / (1 << n)) / np.sqrt(1 << n)
    np.testing.assert_allclose(sv.logical_amplitudes(), want, atol=2e-6)
