"""complex128 5-qubit windows on the tensor cores (tc8d.cu: tcgen05.mma
kind::i8 on seven 8-bit digits per value, levels 0..7 of the digit products
kept, int32 accumulation) against the CPU oracle and against the FP64
CUDA-core kernel (DSV_TC8D=0) on the same inputs.

Bar (north_star): max|d| <= 1e-12 for complex128.  The error is also held
RELATIVE to the amplitude scale to 2e-14 per window — fp64-level (the
CUDA-core FP64 kernel measures ~5e-16 here), so a kernel that silently
dropped a digit level (2^-8 worse per level) fails.
"""

import numpy as np
import pytest

from conftest import assert_state_close, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import _native as N
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu

REL = 2e-14


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


def _apply(st, n, g, tc8d=True):
    N.config_set("tc8d", 1 if tc8d else 0)
    try:
        sv = StateVector.from_amplitudes(st)
        nat = sv.native
        nat.prof_reset()
        nat.prof_enable(True)
        sv.apply(g)
        prof = nat.prof_read()
        nat.prof_enable(False)
        return sv.amplitudes, prof
    finally:
        N.config_set("tc8d", 1)


LAYOUTS = [
    ((0, 1, 2, 3, 4), ()),            # contiguous from bit 0 (tshift)
    ((3, 4, 5, 6, 7), ()),            # contiguous, rows below and above
    ((7, 8, 9, 10, 11), ()),          # contiguous high: rows = bits 0..6
    ((0, 2, 5, 9, 13), ()),           # scattered, bit 0 a target
    ((1, 4, 6, 11, 12), ()),          # scattered, bit 0 free
    ((2, 3, 8, 10, 14), ((0, 1),)),   # control on bit 0
    ((5, 6, 7, 8, 9), ((1, 0), (13, 1))),
]


@pytest.mark.parametrize("targets,controls", LAYOUTS)
def test_tc8d_dense_k5_vs_oracle(targets, controls):
    n = 15
    rng = np.random.default_rng(sum(targets) + 7 * len(controls))
    st = random_state(n, rng, np.complex128)
    g = G.DenseGate(G.random_unitary(32, rng), targets, controls)
    got, prof = _apply(st, n, g)
    assert prof.get("dense_tc", {}).get("count", 0) == 1, prof
    want = st.copy()
    O.apply_gate(want, n, g)
    assert_state_close(got, want, np.complex128)
    rel = np.abs(got - want).max() / np.abs(want).max()
    assert rel <= REL, rel
    fp64, prof64 = _apply(st, n, g, tc8d=False)
    assert "dense_tc" not in prof64
    rel64 = np.abs(fp64 - want).max() / np.abs(want).max()
    assert rel <= max(8 * rel64, 2e-15), (rel, rel64)


def test_tc8d_wide_dynamic_range_and_nonunitary():
    """Rows whose values span many binades, zero rows, and a non-unitary
    (scaled, non-finite-free) matrix: the per-row scale and the gate's
    exponent e_b carry the range."""
    n = 13
    rng = np.random.default_rng(5)
    st = random_state(n, rng, np.complex128)
    st *= np.exp2(rng.integers(-40, 3, st.shape))          # wide dynamic range
    st[rng.integers(0, 1 << n, 64)] = 0
    st[: 1 << 6] = 0                                      # whole groups of zeros
    mat = (rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32))) * 37.5
    g = G.DenseGate(mat, (2, 4, 6, 8, 10), unitary=False)
    got, _ = _apply(st, n, g)
    want = st.copy()
    O.apply_gate(want, n, g)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= REL * scale


def test_tc8d_deep_circuit_matches_fp64():
    """60 windows of k = 5 (QV-like) from a random state: the tensor path
    and the FP64 CUDA-core path agree to 1e-12 and with the oracle."""
    n = 14
    rng = np.random.default_rng(11)
    st = random_state(n, rng, np.complex128)
    gates = [G.DenseGate(G.random_unitary(32, rng), tuple(int(q) for q in rng.permutation(n)[:5]))
             for _ in range(60)]
    want = O.run_circuit(gates, n, state=st)
    outs = []
    for flag in (1, 0):
        N.config_set("tc8d", flag)
        try:
            sv = StateVector.from_amplitudes(st)
            for g in gates:
                sv.apply(g)
            outs.append(sv.amplitudes)
        finally:
            N.config_set("tc8d", 1)
    assert_state_close(outs[0], want, np.complex128)
    assert np.abs(outs[0] - outs[1]).max() <= 1e-13
    assert abs(np.vdot(outs[0], outs[0]).real - 1.0) <= 1e-13


@pytest.mark.parametrize("n", [14, 17])
def test_tc8d_phased_fold_windows(n):
    """The fold fuser's phased 5-qubit windows (pre-phase from unit-factor
    tables per index byte) on tc8d: complex128 QFT from a random state vs the
    oracle and vs the FP64 CUDA-core phased kernel."""
    from paper_2308_01999_b200.circuits import gen_qft, to_gates
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    rng = np.random.default_rng(n)
    st = random_state(n, rng, np.complex128)
    gates = to_gates(gen_qft(n))
    ops = fuse_fold(gates, 5).ops
    outs = []
    for flag in (1, 0):
        N.config_set("tc8d", flag)
        try:
            sv = StateVector.from_amplitudes(st)
            nat = sv.native
            nat.prof_reset()
            nat.prof_enable(True)
            for op in ops:
                sv.apply(op)
            prof = nat.prof_read()
            nat.prof_enable(False)
            outs.append(sv.logical_amplitudes())
            if flag:
                assert prof.get("dense_tc", {}).get("count", 0) >= 2, prof
        finally:
            N.config_set("tc8d", 1)
    want = O.run_circuit(gates, n, state=st)
    assert_state_close(outs[0], want, np.complex128)
    assert np.abs(outs[0] - outs[1]).max() <= 1e-13


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_nonfinite_matrix_propagates_like_numpy(dtype):
    """A non-finite matrix (unitary=False) must not go through the digit
    kernels (they scale by the largest entry): it takes the CUDA cores and
    NaN / inf propagate as in the reference's NumPy product."""
    n = 12
    rng = np.random.default_rng(3)
    st = random_state(n, rng, dtype)
    m = G.random_unitary(32, rng)
    m[3, 7] = np.nan
    g = G.DenseGate(m, (2, 4, 6, 8, 10), unitary=False)
    sv = StateVector.from_amplitudes(st)
    sv.apply(g)
    want = st.astype(np.complex128)
    O.apply_gate(want, n, G.DenseGate(np.asarray(m, dtype=dtype).astype(np.complex128), g.targets, unitary=False))
    got = sv.amplitudes
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    tol = 1e-5 if dtype == np.complex64 else 1e-12
    assert np.abs(got[ok] - want[ok]).max() <= tol
