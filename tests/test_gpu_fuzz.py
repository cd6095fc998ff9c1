"""Seeded fuzzing of the engine against the CPU oracle: random state sizes,
dtypes, gate kinds, arities, target/control layouts, fusers and shardings —
every case a small state the oracle finishes instantly, so the sweep reaches
kernel paths (low-bit, 64-byte-block, warp-transposed, tile, tensor-core,
generic) in combinations the targeted tests do not enumerate.

Bars (BASELINE.json north_star): bit-exact for generalised permutations,
diagonals and index-bit swaps; max |d| <= 1e-5 / 1e-12 (+ relative and
fidelity bars, conftest.assert_state_close) for everything else.
"""

import numpy as np
import pytest

from conftest import assert_state_close, random_state
from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import random_gate_sequence
from paper_2308_01999_b200.statevec import StateVector

pytestmark = pytest.mark.gpu

DTYPES = (np.complex64, np.complex128)


@pytest.fixture(autouse=True)
def _gpu(gpu_available):
    return gpu_available


def _random_gate(n, rng, kmax=6, perm_ok=True):
    k = int(rng.integers(1, min(kmax, n) + 1))
    qs = [int(q) for q in rng.permutation(n)]
    targets = tuple(qs[:k])
    nc = int(rng.integers(0, min(2, n - k) + 1))
    controls = tuple((qs[k + i], int(rng.integers(0, 2))) for i in range(nc))
    kind = int(rng.integers(0, 3)) if perm_ok else 0
    if kind == 0:
        return G.DenseGate(G.random_unitary(1 << k, rng), targets, controls)
    perm = np.arange(1 << k) if kind == 1 else rng.permutation(1 << k)
    return G.PermutationGate(perm, np.exp(1j * rng.uniform(0, 6.3, 1 << k)), targets, controls)


@pytest.mark.parametrize("seed", range(96))
def test_fuzz_single_gates(seed):
    """One random gate on a random state: permutations bit-exact, dense within the bars."""
    rng = np.random.default_rng(1000 + seed)
    for _ in range(6):
        n = int(rng.integers(1, 15))
        dtype = DTYPES[int(rng.integers(0, 2))]
        st = random_state(n, rng, dtype)
        g = _random_gate(n, rng)
        sv = StateVector.from_amplitudes(st)
        sv.apply(g)
        want = st.copy()
        O.apply_gate(want, n, g)
        if isinstance(g, G.PermutationGate):
            np.testing.assert_array_equal(sv.amplitudes, want)
        else:
            ref = st.astype(np.complex128)
            O.apply_gate(ref, n, G.DenseGate(np.asarray(g.matrix, dtype=dtype).astype(np.complex128), g.targets,
                                             g.controls, unitary=False))
            assert_state_close(sv.amplitudes, ref, dtype)


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_circuits_swaps_and_reductions(seed):
    """Random circuits interleaved with index-bit swaps, rotations and
    reductions; the logical state and every reduction against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(3, 15))
    dtype = DTYPES[seed % 2]
    st = random_state(n, rng, dtype)
    sv = StateVector.from_amplitudes(st)
    ref = st.astype(np.complex128)
    for _ in range(10):
        g = _random_gate(n, rng, kmax=5)
        sv.apply(g)
        O.apply_gate(ref, n, g)
        if rng.random() < 0.3:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            sv.swap_index_bits([(a, b)])  # physical relabel: the logical state is unchanged
        if rng.random() < 0.3:
            fac = tuple((int(q), str(rng.choice(list("XYZ")))) for q in rng.permutation(n)[: int(rng.integers(1, n + 1))])
            th = float(rng.uniform(0, 6.3))
            sv.apply_pauli_rotation(th, G.PauliString(fac))
            O.pauli_rotation(ref, n, th, fac)
    got = sv.logical_amplitudes()
    assert_state_close(got, ref, dtype)
    bits = [int(q) for q in rng.permutation(n)[: int(rng.integers(1, min(n, 6) + 1))]]
    tol = 1e-5 if dtype == np.complex64 else 1e-12
    np.testing.assert_allclose(sv.probabilities(bits), O.marginal(ref, n, bits), atol=tol)
    fac = tuple((int(q), str(rng.choice(list("IXYZ")))) for q in rng.permutation(n)[:3])
    assert abs(sv.expectation([G.PauliString(fac)]) - O.expectation_pauli(ref, n, fac)) <= tol
    assert abs(sv.norm_squared() - 1.0) <= 10 * tol


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_fusers_and_shards(seed):
    """Random circuits through the fold and cluster fusers and sharded over
    2/4/8 segments (one device) against the unfused oracle."""
    from paper_2308_01999_b200.fusion_cluster import fuse_cluster
    from paper_2308_01999_b200.fusion_fold import fuse_fold
    from paper_2308_01999_b200.shard import ShardedStateVector

    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(6, 15))
    dtype = DTYPES[seed % 2]
    gates = random_gate_sequence(n, 40, rng, max_arity=3)
    want = O.run_circuit(gates, n)
    k = int(rng.integers(2, 6))
    for ops in (fuse_fold(gates, k).ops, fuse_cluster(gates, k).ops):
        sv = StateVector(n, dtype=dtype)
        for op in ops:
            sv.apply(op)
        assert_state_close(sv.logical_amplitudes(), want, dtype)
    P = int(2 ** rng.integers(1, 4))
    sh = ShardedStateVector(n, [0] * P, dtype)
    sh.run(gates)
    assert_state_close(sh.gather_logical(), want, dtype)
    sh.close()
