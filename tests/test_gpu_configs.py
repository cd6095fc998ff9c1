"""BASELINE configurations and API branches pinned on the B200:

* config 1 (QFT-20 complex128, unfused and FusionConfig(5, 6)) against the
  reference's own outputs (tests/golden/config1.pkl.gz, made by
  oracle/gen_golden.py from the unmodified reference) and against the CPU
  oracle's full state, at the north_star's 1e-12;
* a DEEP complex64 tensor-core workload: fold-fused quantum volume (k = 5
  windows on tcgen05) against the oracle — the int8-digit arithmetic's error
  must not accumulate past the fidelity bar over ~100 windows;
* StateVector.copy and the controlled-DenseGate branch of expectation
  (statevec.py:156-161, :249-252).
"""

import numpy as np
import pytest

from conftest import assert_state_close, fidelity, golden, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, gen_qv, to_gates
from paper_2308_01999_b200.fusion import FusionConfig, fuse
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


@pytest.mark.parametrize("start", ["zero", "random"])
@pytest.mark.parametrize("fused", ["unfused", "fused"])
def test_config1_qft20_c128_vs_reference(start, fused):
    c = golden("config1")
    n = c["n"]
    gates = to_gates(gen_qft(n))
    ops = fuse(gates, FusionConfig(5, 6)).gates if fused == "fused" else gates
    assert len(gates) == c["gates"] and len(fuse(gates, FusionConfig(5, 6)).gates) == c["fused_ops"]
    st = random_state(n, np.random.default_rng(c["state_seed"])) if start == "random" else None
    sv = StateVector.from_amplitudes(st) if st is not None else StateVector(n)
    for g in ops:
        sv.apply(g)
    got = sv.logical_amplitudes()
    ref = c[f"{start}_{fused}"]
    # the reference's own amplitudes (8192 seeded samples), marginals and norm
    assert np.abs(got[c["idx"]] - ref["samples"]).max() <= 1e-12
    np.testing.assert_allclose(sv.probabilities([0, 19, 7, 13]), ref["marginal_0_19_7_13"], atol=1e-12, rtol=0)
    assert abs(sv.norm_squared() - ref["norm"]) <= 1e-12
    # the whole state against the oracle (pinned to the reference)
    want = O.run_circuit(gates, n, state=st)
    assert_state_close(got, want, np.complex128)
    if start == "zero":
        assert np.abs(got - 2.0 ** (-n / 2)).max() <= 1e-12


def test_deep_tensor_core_qv_c64_fidelity():
    """Quantum volume depth 30 at n = 22, fold-fused into k = 5 windows that
    run on the int8-digit tcgen05 kernels, vs the complex128 oracle."""
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 22
    gates = to_gates(gen_qv(n, 30, seed=1))
    ops = fuse_fold(gates, 5).ops
    assert len(ops) >= 60
    st = random_state(n, np.random.default_rng(77), np.complex64)
    sv = StateVector.from_amplitudes(st)
    nat = sv.native
    nat.prof_reset()
    nat.prof_enable(True)
    for op in ops:
        sv.apply(op)
    prof = nat.prof_read()
    nat.prof_enable(False)
    assert prof.get("dense_tc", {}).get("count", 0) >= len(ops) // 2, prof
    want = O.run_circuit(gates, n, dtype=np.complex128, state=st.astype(np.complex128))
    got = sv.logical_amplitudes()
    assert_state_close(got, want, np.complex64)
    assert fidelity(got, want) >= 1 - 1e-6
    assert abs(sv.norm_squared() - 1.0) <= 1e-5


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_copy_is_independent(dtype):
    n = 12
    rng = np.random.default_rng(4)
    st = random_state(n, rng, dtype)
    sv = StateVector.from_amplitudes(st)
    sv.swap_index_bits([(0, 7)])
    cp = sv.copy()
    assert cp.bit_map == sv.bit_map
    np.testing.assert_array_equal(cp.amplitudes, sv.amplitudes)
    cp.apply(G.h(3))
    np.testing.assert_array_equal(sv.logical_amplitudes(), st)
    want = st.copy()
    O.apply_dense(want, n, G.h(3).matrix, [3])
    assert_state_close(cp.logical_amplitudes(), want, dtype)


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_expectation_controlled_dense(dtype):
    """statevec.py:249-252: a DenseGate observable with controls."""
    n = 10
    rng = np.random.default_rng(8)
    st = random_state(n, rng, dtype)
    sv = StateVector.from_amplitudes(st)
    for k, ctrls in ((1, ((4, 1),)), (2, ((0, 0), (9, 1))), (3, ((5, 1),))):
        a = rng.standard_normal((1 << k, 1 << k)) + 1j * rng.standard_normal((1 << k, 1 << k))
        herm = (a + a.conj().T) / 2
        targets = tuple(int(q) for q in rng.permutation([q for q in range(n) if q not in dict(ctrls)])[:k])
        obs = G.DenseGate(herm, targets, ctrls, unitary=False)
        got = sv.expectation(obs)
        want = O.expectation_dense(st.astype(np.complex128), n, herm, list(targets), list(ctrls))
        tol = 1e-5 if dtype == np.complex64 else 1e-12
        assert abs(got - want) <= tol * max(1.0, abs(want))
    np.testing.assert_array_equal(sv.amplitudes, st)
