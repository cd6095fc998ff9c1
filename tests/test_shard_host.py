"""The single-process sharded engine (paper_2308_01999_b200/shard.py) on CPU:
its host protocol — victim choice, batched exchange rounds, segment
relabels, global-control predicates, fold-fuser phase localisation and the
group reductions — driven over a NumPy segment double that implements the
same per-segment primitives as libdsv's NativeState (the exchange as the
masked-pair swap dsv_exchange_pair performs).  The gathered state is checked
against the CPU oracle; the GPU versions of these checks are in
tests/test_gpu_shard.py."""

import itertools

import numpy as np
import pytest

from oracle import sv_oracle as O
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, gen_qv, random_gate_sequence, to_gates
from paper_2308_01999_b200.core import bit_permute_array
from paper_2308_01999_b200.plan import exchange_rounds
from paper_2308_01999_b200.shard import ShardedStateVector


class NumpySeg:
    """Host stand-in for NativeState (one segment)."""

    def __init__(self, nloc, dtype, device):
        self.nloc, self.dtype, self.device = nloc, np.dtype(dtype), device
        self.a = np.zeros(1 << nloc, dtype=self.dtype)
        self.a[0] = 1

    def _groups(self, bits, ctrls):
        idx = np.arange(1 << self.nloc)
        ok = np.ones(idx.size, bool)
        for b, v in ctrls:
            ok &= ((idx >> b) & 1) == v
        for b in bits:
            ok &= ((idx >> b) & 1) == 0
        offs = np.array([sum(((j >> m) & 1) << b for m, b in enumerate(bits)) for j in range(1 << len(bits))])
        return idx[ok][None, :] + offs[:, None]

    def set_zero(self):
        self.a[:] = 0

    def set_basis(self, index=0):
        self.a[:] = 0
        self.a[index] = 1

    def apply_matrix(self, m, bits, ctrls=()):
        g = self._groups(bits, ctrls)
        self.a[g] = np.asarray(m, self.dtype) @ self.a[g]

    def apply_genperm(self, perm, diag, bits, ctrls=()):
        g = self._groups(bits, ctrls)
        out = np.empty_like(self.a[g])
        out[np.asarray(perm)] = np.asarray(diag, self.dtype)[:, None] * self.a[g]
        self.a[g] = out

    def apply_matrix_phased(self, m, bits, cross=(), outside=()):
        idx = np.arange(self.a.size)
        ph = np.zeros(self.a.size)
        for mi, b, t in cross:
            ph += t * (((idx >> bits[mi]) & 1) & ((idx >> b) & 1))
        for b, t in outside:
            ph += t * ((idx >> b) & 1)
        self.a *= np.exp(1j * ph).astype(self.dtype)
        self.apply_matrix(m, bits, [])

    def swap_bits(self, pairs):
        self.a[bit_permute_array(np.arange(self.a.size), pairs)] = self.a.copy()

    def exchange_pair(self, other, lbits, pat_a, pat_b):
        mask = sum(1 << b for b in lbits)
        idx = np.arange(self.a.size)
        off = idx[(idx & mask) == 0]
        x = self.a[off | pat_a].copy()
        self.a[off | pat_a] = other.a[off | pat_b]
        other.a[off | pat_b] = x

    def download(self):
        return self.a.copy()

    def sync(self):
        pass

    def close(self):
        pass

    @staticmethod
    def group_norm2(segs):
        return np.array([float(np.sum(np.abs(s.a) ** 2)) for s in segs])

    @staticmethod
    def group_marginal(segs, bits):
        out = []
        for s in segs:
            idx = np.arange(s.a.size)
            o = np.zeros_like(idx)
            for j, b in enumerate(bits):
                o |= ((idx >> b) & 1) << j
            out.append(np.bincount(o, weights=np.abs(s.a) ** 2, minlength=1 << len(bits)))
        return np.array(out)

    @staticmethod
    def group_expect_pauli(segs, factors):
        out = []
        for s in segs:
            b = s.a.copy()
            idx = np.arange(b.size)
            for bit, p in factors:
                if p in "XY":
                    b = b[idx ^ (1 << bit)]
                    if p == "Y":
                        b = b * np.where((idx >> bit) & 1, 1j, -1j)
                elif p == "Z":
                    b = b * np.where((idx >> bit) & 1, -1, 1)
            out.append(complex(np.vdot(s.a, b)))
        return np.array(out)


def _sharded(n, P, dtype=np.complex128):
    return ShardedStateVector(n, [0] * P, dtype, segment_factory=NumpySeg)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_sharded_circuit_matches_oracle(P):
    n = 7
    rng = np.random.default_rng(5 + P)
    gates = to_gates(gen_qft(n)) + random_gate_sequence(n, 30, rng, max_arity=3)
    gates.append(G.x(6, controls=((5, 1), (4, 0))))
    gates.append(G.DenseGate(G.random_unitary(4, rng), (6, 0), controls=((5, 0),)))
    sv = _sharded(n, P)
    sv.run(gates)
    want = O.run_circuit(gates, n)
    assert np.abs(sv.gather_logical() - want).max() < 1e-12
    assert abs(sv.norm_squared() - 1.0) < 1e-12
    assert np.abs(sv.probabilities([6, 0, 3]) - O.marginal(want, n, [6, 0, 3])).max() < 1e-12
    obs = [G.PauliString(((0, "Z"), (5, "X"), (6, "Y")), 0.5), G.PauliString(((6, "Z"), (1, "Z")))]
    ev = sv.expectation(obs)
    ev_want = sum(O.expectation_pauli(want, n, p.factors, p.coefficient) for p in obs)
    assert abs(ev - ev_want) < 1e-12
    # the relocations for X/Y leave the logical state unchanged
    assert np.abs(sv.gather_logical() - want).max() < 1e-12


@pytest.mark.parametrize("P", [2, 4, 8])
def test_fold_fused_qft_one_reorder(P):
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    n = 8
    sv = _sharded(n, P)
    sv.run(fuse_fold(to_gates(gen_qft(n)), 3).ops)
    assert np.abs(sv.gather_logical() - O.run_circuit(to_gates(gen_qft(n)), n)).max() < 1e-12
    # |0> placement puts the last-targeted qubits on the global bits: one reorder
    assert sv.stats.num_reorders == 1


@pytest.mark.parametrize("P,pairs", [
    (2, [(6, 0)]), (2, [(6, 3), (1, 2)]), (4, [(6, 0), (5, 2)]), (4, [(5, 1), (6, 4), (0, 3)]),
    (8, [(4, 0), (5, 1), (6, 2)]), (8, [(6, 4), (5, 0)]), (8, [(6, 5)]), (4, [(6, 5), (0, 1)]),
])
def test_distributed_swap_equals_full_vector_swap(P, pairs):
    n = 7
    rng = np.random.default_rng(1)
    full = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n))
    sv = _sharded(n, P)
    nloc = sv.local_bits
    for s, seg in enumerate(sv.segs):
        seg.a[:] = full[s << nloc:(s + 1) << nloc]
    sv.distributed_index_bit_swap(pairs)
    got = np.concatenate([seg.a for seg in sv.segs])
    want = np.empty_like(full)
    want[bit_permute_array(np.arange(full.size), pairs)] = full
    assert np.array_equal(got, want)


@pytest.mark.parametrize("q,g", [(1, 1), (1, 3), (2, 2), (2, 3), (3, 3)])
def test_exchange_rounds_are_perfect_matchings(q, g):
    nseg = 1 << g
    gl = [(j, 10 + j) for j in range(q)]
    rounds = {}
    for m, s, t, lbits, ps, pt in exchange_rounds(gl, nseg):
        rounds.setdefault(m, []).append((s, t))
        assert lbits == [10 + j for j in range(q)]
    assert len(rounds) == (1 << q) - 1
    for pairs in rounds.values():
        members = list(itertools.chain(*pairs))
        assert sorted(members) == list(range(nseg))


def test_sharded_qv_c64_p_invariant_on_host():
    """Group arithmetic does not depend on the layout: the same op sequence
    on 2 and 4 segments gives bit-identical states (the GPU form of this
    check is the P-invariance test in tests/test_gpu_shard.py)."""
    n = 8
    gates = to_gates(gen_qv(n, 6, seed=2))
    outs = []
    for P in (2, 4):
        sv = _sharded(n, P, np.complex64)
        sv.run(gates)
        outs.append(sv.gather_logical())
    assert np.abs(outs[0] - outs[1]).max() < 1e-5
