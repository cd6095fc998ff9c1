"""Tensor-core dense path on the B200 against the CPU oracle.

Complex64 dense / phased windows of k = 4, 5 (and 6, tc68.cu) run on
tcgen05: by default the int8-digit kernels (tc8.cu: tcgen05.mma kind::i8 on
exact 8-bit digits, int32 accumulation, A operand in TMEM — the two-group
kernel with per-thread cp.async or TMA tile loads, and the warp-specialised
pipeline), with DSV_TC8=0 the bf16-limb kernels (tc.cu / tc6.cu, kind::f16).
Bar (north_star): max|d| <= 1e-5 for complex64; the error is also held
RELATIVE to the amplitude scale to 5e-6 (the int8 digits drop products below
2^-22 of the row scale: ~1.5e-6 per window), so a silently degraded 1-pass
TF32 / bf16 product (~5e-4) fails.
"""

import numpy as np
import pytest

from conftest import random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import _native as N
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu

REL = 5e-6


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


def _rel_err(got, want):
    return float(np.abs(got - want).max() / np.abs(want).max())


def _phase_angles(n, targets, cross, outside):
    """Per-amplitude pre-phase of a phased window (fusion_fold.PhasedDenseGate):
    sum t * x_targets[m] * x_b over cross terms + sum t * x_b over outside terms."""
    idx = np.arange(1 << n, dtype=np.int64)
    ang = np.zeros(1 << n)
    for m, b, t in cross:
        ang += t * (((idx >> targets[m]) & 1) * ((idx >> b) & 1))
    for b, t in outside:
        ang += t * ((idx >> b) & 1)
    return ang


def _tc_launches(sv):
    nat = sv.native
    nat.prof_enable(True)
    nat.prof_reset()
    return nat


@pytest.mark.parametrize("k", [5])
def test_tc_dense_vs_oracle(k):
    rng = np.random.default_rng(900 + k)
    for trial in range(6):
        n = int(rng.integers(k + 8, 19))
        pool = list(range(2, n))
        targets = [int(x) for x in rng.choice(pool, size=k, replace=False)]
        rest = [q for q in range(1, n) if q not in targets]  # bit 0 stays free (16-byte row pairs)
        ctrls = [(int(q), int(rng.integers(0, 2))) for q in rng.permutation(rest)[: trial % 3]]
        if n - k - len(ctrls) < 7:
            ctrls = []
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng)
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, ctrls)
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
        prof = nat.prof_read()
        assert prof.get("dense_tc", {}).get("count", 0) == 1, prof
        got = sv.amplitudes
        assert np.abs(got - want).max() <= 1e-5
        assert _rel_err(got, want) <= REL, (trial, targets, ctrls, _rel_err(got, want))


@pytest.mark.parametrize("k", [4, 5, 6])
@pytest.mark.parametrize("scale", [2.0 ** -12, 0.37, 3.1, 2.0 ** 9])
def test_tc_scaled_matrices_and_tiny_states(k, scale):
    """Non-unitary (scaled) gate matrices move the gate exponent e_b; a state
    scaled by 2^-60 moves every row exponent: the digit scaling must follow
    both (relative error unchanged)."""
    rng = np.random.default_rng(int(1000 * scale) + k)
    n = 16
    targets = list(range(4, 4 + k)) if k != 4 else [0, 1, 2, 3]
    m = (G.random_unitary(1 << k, rng) * scale).astype(np.complex64)
    for amp_scale in (1.0, 2.0 ** -60):
        st = (random_state(n, rng, np.complex64) * np.float32(amp_scale)).astype(np.complex64)
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m.astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.apply_matrix(G.DenseGate(m, tuple(targets), unitary=False))
        assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
        assert _rel_err(sv.amplitudes, want) <= 2 * REL, (amp_scale, _rel_err(sv.amplitudes, want))


@pytest.mark.parametrize("case", ["low0", "low0c", "bit1", "ctrl0", "spread0"])
def test_tc_dense_low_bits_vs_oracle(case):
    """Index bit 0 a target or control: the 8-byte-per-row (non-pair) copies."""
    rng = np.random.default_rng(hash(case) % 1000)
    n = 16
    targets, ctrls = {
        "low0": ([0, 1, 2, 3, 4], []),         # contiguous tiles (row-major staging)
        "low0c": ([0, 1, 2, 3, 4], [(13, 1)]),
        "bit1": ([1, 2, 3, 9, 14], []),
        "ctrl0": ([2, 5, 8, 11, 15], [(0, 1)]),
        "spread0": ([0, 4, 7, 10, 13], [(15, 0)]),
    }[case]
    targets = [int(t) for t in rng.permutation(targets)]
    st = random_state(n, rng, np.complex64)
    m = G.random_unitary(32, rng)
    want = st.astype(np.complex128)
    O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, ctrls)
    sv = StateVector.from_amplitudes(st)
    nat = _tc_launches(sv)
    sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
    assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
    assert _rel_err(sv.amplitudes, want) <= REL


@pytest.mark.parametrize("targets,ctrls", [([0, 5, 9, 14], []), ([0, 2, 3, 4], []),
                                           ([0, 6, 7, 8], [(12, 1)]), ([0, 3, 10, 15], [(13, 0)])])
def test_tc_k4_bit0_target_vs_oracle(targets, ctrls):
    """Plain k = 4 with index bit 0 a target takes the tensor path (16-byte
    member pairs); every other k = 4 layout except bits 0..3 stays on the CUDA cores."""
    rng = np.random.default_rng(sum(targets))
    n = 16
    targets = [int(t) for t in rng.permutation(targets)]
    st = random_state(n, rng, np.complex64)
    m = G.random_unitary(16, rng)
    want = st.astype(np.complex128)
    O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, ctrls)
    sv = StateVector.from_amplitudes(st)
    nat = _tc_launches(sv)
    sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
    assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
    assert np.abs(sv.amplitudes - want).max() <= 1e-5
    assert _rel_err(sv.amplitudes, want) <= REL
    sv2 = StateVector.from_amplitudes(st)
    nat = _tc_launches(sv2)
    sv2.apply_matrix(G.DenseGate(m, (1, 5, 9, 14)))
    assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 0  # bit 0 free: CUDA cores


@pytest.mark.parametrize("k", [4, 5])
def test_tc_phased_vs_oracle(k):
    rng = np.random.default_rng(950 + k)
    for trial in range(4):
        n = int(rng.integers(k + 8, 19))
        targets = [int(x) for x in rng.choice(np.arange(2, n), size=k, replace=False)]
        if trial == 3:
            targets[0] = 0  # index bit 0 a target: per-row copies
        if trial == 2:
            targets = list(range(k))  # the lowest k bits: contiguous tiles
        outside_bits = [q for q in range(n) if q not in targets]
        cross = [(int(rng.integers(0, k)), int(b), float(rng.uniform(-7, 7)))
                 for b in rng.choice(outside_bits, size=min(12, len(outside_bits)), replace=False)]
        outside = [(int(b), float(rng.uniform(-7, 7))) for b in rng.choice(outside_bits, size=5, replace=False)]
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng).astype(np.complex64)
        want = st.astype(np.complex128) * np.exp(1j * _phase_angles(n, targets, cross, outside))
        O.apply_dense(want, n, m.astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.native.apply_matrix_phased(m, targets, cross, outside)
        sv._mutated()
        prof = nat.prof_read()
        assert prof.get("dense_tc", {}).get("count", 0) == 1, prof
        got = sv.amplitudes
        # float32 angle tables + fast sincos: ~1e-6 phase error on top of the product
        assert _rel_err(got, want) <= 2 * REL, (trial, _rel_err(got, want))


@pytest.mark.parametrize("nrow", [0, 1, 2, 3, 4])
def test_tc_phased_row_vectors_vs_oracle(nrow):
    """Phase terms on 0..4 of a tile's row bits (the 7 lowest free bits) plus
    tile-uniform bits: <= 3 row bits take the per-tile phase-vector path of
    tc8.cu, 4 the per-row path — both against the oracle."""
    rng = np.random.default_rng(1200 + nrow)
    k = 5
    for trial in range(3):
        n = int(rng.integers(14, 19))
        t0 = int(rng.integers(3, n - k - 2)) if trial != 2 else 1
        targets = list(range(t0, t0 + k))
        free = [q for q in range(n) if q not in targets]
        rowbits, uniform = free[:7], free[7:]
        pick = [int(b) for b in rng.choice(rowbits, size=nrow, replace=False)] if nrow else []
        bits = pick + [int(b) for b in rng.choice(uniform, size=min(4, len(uniform)), replace=False)]
        cross = [(int(rng.integers(0, k)), b, float(rng.uniform(-7, 7))) for b in bits for _ in range(2)]
        outside = [(b, float(rng.uniform(-7, 7))) for b in bits]
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng).astype(np.complex64)
        want = st.astype(np.complex128) * np.exp(1j * _phase_angles(n, targets, cross, outside))
        O.apply_dense(want, n, m.astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.native.apply_matrix_phased(m, targets, cross, outside)
        sv._mutated()
        assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
        assert _rel_err(sv.amplitudes, want) <= 2 * REL, (trial, _rel_err(sv.amplitudes, want))


def test_tc_involution_round_trip_large():
    """U then U^dagger on a 24-qubit state with a target in every position
    class (low/mid/high): returns the input to fp32-level accuracy."""
    rng = np.random.default_rng(77)
    n = 24
    st = random_state(n, rng, np.complex64)
    sv = StateVector.from_amplitudes(st)
    for targets in ([2, 3, 4, 5, 6], [7, 11, 13, 17, 23], [19, 20, 21, 22, 23], [2, 9, 15, 22]):
        m = G.random_unitary(1 << len(targets), rng)
        sv.apply_matrix(G.DenseGate(m, tuple(targets)))
        sv.apply_matrix(G.DenseGate(m.conj().T, tuple(targets)))
    got = sv.amplitudes
    assert _rel_err(got, st) <= 4 * REL
    fid = abs(np.vdot(st.astype(np.complex128), got.astype(np.complex128))) ** 2
    assert fid >= 1 - 1e-6


def test_tc_tail_tiles_and_grid_stride():
    """nwork = 2^(n-k) from exactly one 128-group tile up to many tiles per CTA."""
    rng = np.random.default_rng(5)
    for n in (12, 13, 20):
        k = 5
        targets = list(range(n - k, n))  # high targets: groups = low free bits
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng)
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        sv.apply_matrix(G.DenseGate(m, tuple(targets)))
        assert _rel_err(sv.amplitudes, want) <= REL


# ---- lane-split kernel: k <= 3 windows on the lowest k bits (low.cu) ------------------------

@pytest.mark.parametrize("k", [2, 3])
def test_low_dense_vs_oracle(k):
    rng = np.random.default_rng(700 + k)
    for trial in range(4):
        n = int(rng.integers(14, 19))  # >= 1024 lane-items: whole passes
        targets = [int(x) for x in rng.permutation(k)]  # bits 0..k-1, any order
        rest = list(range(k, n))
        ctrls = [(int(q), int(rng.integers(0, 2))) for q in rng.permutation(rest)[: trial % 3]]
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng)
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, ctrls)
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
        # uncontrolled windows inside bits 0..2 take the 64-byte-block kernel (perm.cu k_dense_blk8)
        want_cls = "dense_low" if ctrls else "dense"
        assert nat.prof_read().get(want_cls, {}).get("count", 0) == 1
        assert _rel_err(sv.amplitudes, want) <= 1e-6


@pytest.mark.parametrize("k", [1, 2, 3])
def test_low_phased_vs_oracle(k):
    rng = np.random.default_rng(750 + k)
    for trial in range(3):
        n = int(rng.integers(12, 19))
        targets = list(range(k))
        outside_bits = list(range(k, n))
        cross = [(int(rng.integers(0, k)), int(b), float(rng.uniform(-7, 7)))
                 for b in rng.choice(outside_bits, size=min(14, len(outside_bits)), replace=False)]
        outside = [(int(b), float(rng.uniform(-7, 7))) for b in rng.choice(outside_bits, size=4, replace=False)]
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(1 << k, rng).astype(np.complex64)
        want = st.astype(np.complex128) * np.exp(1j * _phase_angles(n, targets, cross, outside))
        O.apply_dense(want, n, m.astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.native.apply_matrix_phased(m, targets, cross, outside)
        sv._mutated()
        assert nat.prof_read().get("dense_low", {}).get("count", 0) == 1
        assert _rel_err(sv.amplitudes, want) <= 2 * REL, (trial, _rel_err(sv.amplitudes, want))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_low_phased_complex128_vs_oracle(k):
    """complex128 windows on the lowest k bits (warp-transposed runs with the
    unit-factor phase tables), plain and phased, against the oracle."""
    rng = np.random.default_rng(1750 + k)
    for trial in range(3):
        n = int(rng.integers(12, 17))
        targets = list(range(k))
        outside_bits = list(range(k, n))
        if trial == 0:
            cross, outside = [], []
        else:
            cross = [(int(rng.integers(0, k)), int(b), float(rng.uniform(-7, 7)))
                     for b in rng.choice(outside_bits, size=min(12, len(outside_bits)), replace=False)]
            outside = [(int(b), float(rng.uniform(-7, 7))) for b in rng.choice(outside_bits, size=4, replace=False)]
        st = random_state(n, rng, np.complex128)
        m = G.random_unitary(1 << k, rng)
        want = st * np.exp(1j * _phase_angles(n, targets, cross, outside))
        O.apply_dense(want, n, m, targets, [])
        sv = StateVector.from_amplitudes(st)
        sv.native.apply_matrix_phased(m, targets, cross, outside)
        sv._mutated()
        assert _rel_err(sv.amplitudes, want) <= 1e-12, (trial, _rel_err(sv.amplitudes, want))


# ---- k = 6 windows (tc6.cu) -------------------------------------------------------------------

@pytest.mark.parametrize("case", ["high", "mid", "spread", "bit0", "ctrl", "bits01", "low6", "bit1", "bit0ctrl"])
def test_tc6_dense_vs_oracle(case):
    rng = np.random.default_rng(600 + len(case))
    n = 17
    targets, ctrls = {
        "high": (list(range(11, 17)), []),
        "mid": ([4, 5, 6, 7, 8, 9], []),
        "spread": ([2, 5, 8, 11, 13, 16], []),
        "bit0": ([0, 3, 6, 9, 12, 15], []),        # per-row 8-byte copies
        "ctrl": ([3, 6, 7, 9, 12, 14], [(16, 1)]),
        "bits01": ([0, 1, 4, 7, 9, 12], []),       # both low bits targets (formerly the generic kernel)
        "low6": ([0, 1, 2, 3, 4, 5], []),          # contiguous low window, per-row copies
        "bit1": ([1, 3, 5, 8, 10, 12], []),        # member-parity lanes + pair-swapped stores
        "bit0ctrl": ([0, 3, 6, 9, 12, 14], [(16, 1)]),  # row2 with a control
    }[case]
    targets = [int(t) for t in rng.permutation(targets)]
    st = random_state(n, rng, np.complex64)
    m = G.random_unitary(64, rng)
    want = st.astype(np.complex128)
    O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), targets, ctrls)
    sv = StateVector.from_amplitudes(st)
    nat = _tc_launches(sv)
    sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
    assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
    assert _rel_err(sv.amplitudes, want) <= REL, _rel_err(sv.amplitudes, want)


def test_tc6_phased_and_fold_qft():
    rng = np.random.default_rng(66)
    n = 16
    for targets in ([2, 4, 6, 8, 10, 12], [10, 11, 12, 13, 14, 15]):
        outside_bits = [q for q in range(n) if q not in targets]
        cross = [(int(rng.integers(0, 6)), int(b), float(rng.uniform(-7, 7)))
                 for b in rng.choice(outside_bits, size=8, replace=False)]
        outside = [(int(b), float(rng.uniform(-7, 7))) for b in rng.choice(outside_bits, size=3, replace=False)]
        st = random_state(n, rng, np.complex64)
        m = G.random_unitary(64, rng).astype(np.complex64)
        want = st.astype(np.complex128) * np.exp(1j * _phase_angles(n, targets, cross, outside))
        O.apply_dense(want, n, m.astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        sv.native.apply_matrix_phased(m, targets, cross, outside)
        sv._mutated()
        assert _rel_err(sv.amplitudes, want) <= 2 * REL
    # folded QFT at k = 6 (tensor-core 6-qubit windows) = DFT column
    from paper_2308_01999_b200.circuits import gen_qft, to_gates
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n, x = 18, 54321
    st = np.zeros(1 << n, np.complex64)
    st[x] = 1
    sv = StateVector.from_amplitudes(st)
    for op in fuse_fold(to_gates(gen_qft(n)), 6).ops:
        sv.apply(op)
    y = np.arange(1 << n)
    dft = np.exp(2j * np.pi * x * y / (1 << n)) / np.sqrt(1 << n)
    assert np.abs(sv.logical_amplitudes() - dft).max() < 2e-6


def test_phased_k6_off_tensor_path_falls_back():
    """Complex128 (no tensor path): the host applies the phases as diagonals."""
    from paper_2308_01999_b200.circuits import gen_qft, to_gates
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 12
    st = np.zeros(1 << n, np.complex128)
    st[77] = 1
    sv = StateVector.from_amplitudes(st)
    for op in fuse_fold(to_gates(gen_qft(n)), 6).ops:
        sv.apply(op)
    y = np.arange(1 << n)
    dft = np.exp(2j * np.pi * 77 * y / (1 << n)) / np.sqrt(1 << n)
    assert np.abs(sv.logical_amplitudes() - dft).max() < 1e-12


# ---- warp-transpose kernel: dense gates inside the lowest 6 bits (wt.cu) --------------------

@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_wt_low_targets_vs_oracle(dtype):
    rng = np.random.default_rng(31)
    n = 14
    cases = [[1, 2, 3], [1, 3, 5], [2, 4]] if dtype == np.complex64 else [[0, 1, 2], [0, 2], [1, 2, 5], [0, 1, 2, 3]]
    for targets in cases:
        targets = [int(t) for t in rng.permutation(targets)]
        st = random_state(n, rng, dtype)
        m = G.random_unitary(1 << len(targets), rng)
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m.astype(dtype).astype(np.complex128), targets, [])
        sv = StateVector.from_amplitudes(st)
        nat = _tc_launches(sv)
        sv.apply_matrix(G.DenseGate(m, tuple(targets)))
        prof = nat.prof_read()
        if sorted(targets) in ([1, 2, 3], [0, 1, 2], [0, 1, 2, 3]):
            assert prof.get("dense_wt", {}).get("count", 0) == 1, prof
        tol = 2e-6 if dtype == np.complex64 else 1e-13
        assert _rel_err(sv.amplitudes, want) <= tol, (targets, prof, _rel_err(sv.amplitudes, want))


@pytest.mark.parametrize("targets", [(5, 6, 7, 8, 9), (2, 9, 15, 3, 12), (1, 4, 6, 9, 12), (0, 5, 9, 12, 14),
                                     (0, 1, 2, 3, 4), (0, 1, 2, 3), (0, 2, 5, 7)])
def test_tc8_kernel_variants_all_layouts(targets):
    """Every int8-digit kernel variant forced on for every copy mode, plain and
    phased, against the oracle: the warp-specialised pipeline (tc8.cu
    k_dense_tc8ws: loader / converter / epilogue warps), the two-group kernel
    with per-thread cp.async copies, and the two-group kernel with TMA tile
    loads (cp.async.bulk.tensor, mode kTcTma, where the layout allows)."""
    from paper_2308_01999_b200.fusion_fold import PhasedDenseGate

    rng = np.random.default_rng(sum(targets) + 31 * len(targets))
    n = 16
    k = len(targets)
    m = G.random_unitary(1 << k, rng)
    others = [q for q in range(n) if q not in targets]
    cross = tuple((int(targets[i]), int(others[(3 * i) % len(others)]), float(rng.uniform(0, 6))) for i in range(k))
    outside = ((int(others[-1]), 0.7),)
    st = random_state(n, rng, np.complex64)
    for op in (G.DenseGate(m, tuple(targets)), PhasedDenseGate(m, tuple(targets), cross, outside)):
        want = st.astype(np.complex128)
        if isinstance(op, PhasedDenseGate):
            ang = _phase_angles(n, list(range(n)), [(q, b, t) for q, b, t in cross], list(outside))
            want = want * np.exp(1j * ang)
        O.apply_dense(want, n, m, list(targets))
        outs = []
        for ws, tma in ((1, 1), (0, 0), (0, 1)):
            N.config_set("tc8ws", ws)
            N.config_set("tma", tma)
            try:
                sv = StateVector.from_amplitudes(st)
                nat = _tc_launches(sv)
                sv.apply(op)
                assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1
                outs.append(sv.amplitudes)
            finally:
                N.config_set("tc8ws", 1)
                N.config_set("tma", 1)
        for o in outs:
            assert _rel_err(o, want) <= 2 * REL


# ---- routing added in round 2: layouts that formerly took the CUDA-core or generic kernels ----

@pytest.mark.parametrize("targets", [
    (3, 4, 5, 6), (8, 9, 10, 11),                 # k = 4, contiguous from bit 3 up -> tensor cores
    (0, 1, 4, 7), (0, 1, 6, 9, 12), (0, 1, 2, 7, 11),   # targets on bits 0 and 1 (member-pair mode)
    (0, 1, 4, 7, 9, 12), (0, 2, 5, 8, 10, 13),   # k = 6 with bit 0 a target (tc68 row2)
])
@pytest.mark.parametrize("ctrls", [(), ((14, 1),)])
def test_round2_tensor_routing_vs_oracle(targets, ctrls):
    n = 15
    if ctrls and len(targets) == 4 and targets[0] >= 3:
        pytest.skip("controlled k = 4 gates stay on the CUDA cores")
    rng = np.random.default_rng(sum(targets) + 31 * len(targets))
    st = random_state(n, rng, np.complex64)
    m = G.random_unitary(1 << len(targets), rng)
    want = st.astype(np.complex128)
    O.apply_dense(want, n, m.astype(np.complex64).astype(np.complex128), list(targets), list(ctrls))
    sv = StateVector.from_amplitudes(st)
    nat = _tc_launches(sv)
    sv.apply_matrix(G.DenseGate(m, tuple(targets), tuple(ctrls)))
    assert nat.prof_read().get("dense_tc", {}).get("count", 0) == 1, nat.prof_read()
    assert _rel_err(sv.amplitudes, want) <= REL, _rel_err(sv.amplitudes, want)
