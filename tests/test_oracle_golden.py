"""Pin the CPU oracle (oracle/sv_oracle.py) against golden vectors produced by
the reference package itself (oracle/gen_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import gate_from_spec, golden
from oracle import sv_oracle as O

DT = {"complex64": np.complex64, "complex128": np.complex128}


def _exact_or_close(got, want, dtype, exact):
    if exact:
        np.testing.assert_array_equal(got, want)
    else:
        tol = 1e-5 if dtype == "complex64" else 1e-12
        np.testing.assert_allclose(got, want, atol=tol, rtol=0)


def test_single_ops_match_reference():
    for case in golden("single_ops"):
        g = gate_from_spec(case["gate"])
        amps = case["in"].copy()
        O.apply_gate(amps, case["n"], g)
        # generalised permutations are bit-exact (NumPy FMA-form product)
        _exact_or_close(amps, case["out"], case["dtype"], exact=case["gate"]["kind"] == "perm")


def test_random_circuits_match_reference():
    for case in golden("sv_random"):
        gates = [gate_from_spec(s) for s in case["gates"]]
        out = O.run_circuit(gates, case["n"], dtype=DT[case["dtype"]])
        _exact_or_close(out, case["out"], case["dtype"], exact=False)


def test_swap_and_access_match_reference():
    for c in golden("swap_access"):
        n = c["n"]
        out = O.swap_index_bits(c["in"], n, c["pairs"])
        np.testing.assert_array_equal(out, c["out"])
        np.testing.assert_array_equal(O.access(out, n, c["ordering"], c["begin"], c["end"]), c["access"])
        logical = O.access(out, n, c["bit_map"])
        np.testing.assert_array_equal(logical, c["logical"])
        amps = c["in"].copy()
        O.access_set(amps, n, c["ordering"], c["begin"], c["set_values"])
        np.testing.assert_array_equal(amps, c["after_set"])


def test_measure_expectation_sample_match_reference():
    for c in golden("measure"):
        n, st = c["n"], c["in"]
        np.testing.assert_allclose(O.marginal(st, n, c["qubits"]), c["probs"], rtol=1e-6, atol=1e-7)
        outcome, collapsed = O.measure(st, n, c["qubits"], c["r"])
        assert outcome == c["outcome"]
        np.testing.assert_allclose(collapsed, c["collapsed"], atol=1e-6)
        ev = sum(O.expectation_pauli(st, n, f, coef) for f, coef in c["paulis"])
        assert abs(ev - c["ev_pauli"]) < 1e-5
        evd = O.expectation_dense(st, n, c["herm"], c["herm_targets"])
        assert abs(evd - c["ev_dense"]) < 1e-5
        rot = st.copy()
        O.pauli_rotation(rot, n, c["theta"], c["rot"][0], c["rot"][1])
        np.testing.assert_allclose(rot, c["rotated"], atol=1e-6)
        idx = O.sample_indices(st, len(c["shots"]), c["seed"])
        order = c["order"] if c["order"] is not None else list(range(n - 1, -1, -1))
        strings = ["".join(str((int(i) >> b) & 1) for b in order) for i in idx]
        assert strings == c["shots"]


def test_qft_states_match_reference():
    from paper_2308_01999_b200.circuits import gen_qft, to_gates

    for n, want in golden("misc")["qft_states"].items():
        got = O.run_circuit(to_gates(gen_qft(n)), n)
        np.testing.assert_allclose(got, want, atol=1e-12)


def test_full_operator_agrees_with_kernel_restatement():
    rng = np.random.default_rng(3)
    for case in golden("single_ops")[:40]:
        n = case["n"]
        if n > 7:
            continue
        g = gate_from_spec(case["gate"])
        mat = g.matrix if case["gate"]["kind"] == "dense" else g.to_matrix()
        full = O.full_operator(n, mat, g.targets, g.controls)
        want = full @ case["in"].astype(np.complex128)
        tol = 1e-5 if case["dtype"] == "complex64" else 1e-12
        np.testing.assert_allclose(case["out"], want, atol=tol)
    assert rng is not None


@pytest.mark.parametrize("pairs", [[(0, 7), (2, 9), (4, 5)], [(1, 3)], [(0, 9)]])
def test_bit_permute_naive(pairs):
    from paper_2308_01999_b200.core import bit_permute

    m = golden("misc")["bit_permute"]
    for x, y in zip(m["x"], m["y"]):
        assert O.bit_permute_naive(int(x), m["pairs"]) == y
    for x in range(1 << 10):
        assert bit_permute(x, pairs) == O.bit_permute_naive(x, pairs)


def test_config1_qft20_matches_reference():
    """BASELINE config 1 (QFT-20 complex128, unfused 220 gates and fused
    (5, 6) 66 ops) from |0> and a seeded random state: the oracle reproduces
    the reference's sampled amplitudes, marginals and norm."""
    from conftest import random_state
    from paper_2308_01999_b200.circuits import gen_qft, to_gates
    from paper_2308_01999_b200.fusion import FusionConfig, fuse

    c = golden("config1")
    n = c["n"]
    gates = to_gates(gen_qft(n))
    fused = fuse(gates, FusionConfig(5, 6)).gates
    for start in ("zero", "random"):
        st = random_state(n, np.random.default_rng(c["state_seed"])) if start == "random" else None
        for tag, ops in (("unfused", gates), ("fused", fused)):
            a = O.run_circuit(ops, n, state=st)
            ref = c[f"{start}_{tag}"]
            assert np.abs(a[c["idx"]] - ref["samples"]).max() <= 1e-13
            np.testing.assert_allclose(O.marginal(a, n, [0, 19, 7, 13]), ref["marginal_0_19_7_13"], atol=1e-13)
