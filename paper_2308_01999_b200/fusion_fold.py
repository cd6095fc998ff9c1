"""Opt-in gate fusion with phase folding.

The reference fuser (fusion.py, kept bit-for-bit for drop-in parity) fuses
QFT-33 into 152 windows, 119 of them diagonal.  On a B200 every window is a
full HBM pass, so the window count IS the runtime.  This fuser removes the
diagonal passes:

* Every <= 2-qubit unit-modulus diagonal (CP, CZ, RZ, RZZ, P, S, T, Z, any
  controlled phase) is a degree-<=2 phase polynomial
      exp(i (c + t_a x_a + t_b x_b + t_ab x_a x_b)).
* "Matrix" gates (everything else) are packed greedily into dense windows of
  <= k qubits, scanning the whole remaining circuit and pulling gates
  forward past gates they commute with (disjoint qubits, or both diagonal).
* A phase gate is folded into the window that first acts on one of its
  qubits: fully inside -> multiplied into the window matrix in circuit
  order; one qubit a inside (and not yet acted on), the other b outside ->
  a *cross term* t_ab x_a x_b of the window's pre-phase, evaluated per
  amplitude group on the GPU from b's bit (dsv_apply_matrix_phased); a
  linear term on an outside qubit becomes an outside term.
* SWAP gates become qubit relabels (no data movement): the StateVector's
  bit_map absorbs them, ``logical_amplitudes()`` is unchanged.
* Phase gates that no later matrix gate touches are packed into diagonal
  windows (<= max_fused_diagonal_gate_size qubits) at the end.

QFT-33 with k = 5 becomes 7 phased dense passes (+ relabels).  Results equal
the unfused circuit to floating-point tolerance (tests/test_fusion_fold.py).
"""

from __future__ import annotations

import cmath
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from .core import InvalidArgumentError
from .fusion import _fused_diagonal, expand_gate
from .gates import DenseGate, Gate, PermutationGate


@dataclass
class PhasedDenseGate:
    """Dense matrix on ``targets`` applied after the diagonal
    exp(i (sum_{(a,b,t)} t x_a x_b + sum_{(b,t)} t x_b)) where a is a target
    qubit and b a qubit outside the window."""

    matrix: np.ndarray
    targets: tuple[int, ...]
    cross: list[tuple[int, int, float]] = field(default_factory=list)
    outside: list[tuple[int, float]] = field(default_factory=list)
    controls: tuple = ()

    @property
    def qubits(self) -> tuple[int, ...]:
        return self.targets + tuple(b for _, b, _ in self.cross) + tuple(b for b, _ in self.outside)


@dataclass
class QubitSwap:
    """SWAP(a, b) realised as a relabel of the logical->physical bit map."""

    a: int
    b: int

    @property
    def qubits(self) -> tuple[int, ...]:
        return (self.a, self.b)


@dataclass
class FoldedCircuit:
    ops: list
    provenance: list[list[int]]

    def __len__(self) -> int:
        return len(self.ops)

    @property
    def data_passes(self) -> int:
        return sum(1 for op in self.ops if not isinstance(op, QubitSwap))


@dataclass
class _Phase:
    qubits: tuple[int, ...]      # 1 or 2 qubits
    const: float
    lin: dict[int, float]
    quad: float                  # coefficient of x_q0 x_q1 (2-qubit only)


def _phase_poly(g: Gate) -> _Phase | None:
    """Phase-polynomial form of a <= 2-qubit unit-modulus diagonal, else None."""
    if not isinstance(g, PermutationGate):
        return None
    qs = list(g.targets) + [q for q, _ in g.controls]
    if len(qs) > 2:
        return None
    # tiny tables: Python scalars beat NumPy's per-call overhead (577 gates per QFT-33)
    perm = g.permutation.tolist()
    if perm != list(range(len(perm))):
        return None
    diag = g.diagonal.tolist()
    if any(abs(abs(z) - 1.0) > 1e-12 for z in diag):
        return None
    pos = {q: i for i, q in enumerate(qs)}

    def entry(x: int) -> complex:  # x: bit i = value of qs[i]
        for q, v in g.controls:
            if ((x >> pos[q]) & 1) != v:
                return 1.0
        j = 0
        for m, q in enumerate(g.targets):
            j |= ((x >> pos[q]) & 1) << m
        return diag[j]

    if len(qs) == 1:
        c = cmath.phase(entry(0))
        return _Phase((qs[0],), c, {qs[0]: cmath.phase(entry(1)) - c}, 0.0)
    e00, e10, e01, e11 = (cmath.phase(entry(x)) for x in (0, 1, 2, 3))
    return _Phase((qs[0], qs[1]), e00, {qs[0]: e10 - e00, qs[1]: e01 - e00}, e11 - e10 - e01 + e00)


def _is_swap(g: Gate) -> bool:
    return (isinstance(g, PermutationGate) and not g.controls and len(g.targets) == 2
            and g.permutation.tolist() == [0, 2, 1, 3] and g.diagonal.tolist() == [1, 1, 1, 1])


def _diag_gate(qubits, const: float, lin: dict, quad: float) -> PermutationGate:
    """Diagonal PermutationGate of a phase polynomial on ``qubits``."""
    qs = list(qubits)
    d = np.empty(1 << len(qs), dtype=np.complex128)
    for x in range(d.size):
        ph = const + sum(t for q, t in lin.items() if (x >> qs.index(q)) & 1)
        if len(qs) == 2 and (x & 3) == 3:
            ph += quad
        d[x] = cmath.exp(1j * ph)
    return PermutationGate(np.arange(d.size), d, tuple(qs))


def fuse_fold(circuit: Sequence[Gate], max_gate_size: int = 5, max_diag_size: int = 10,
              relabel_swaps: bool = True) -> FoldedCircuit:
    ops: list = []
    prov: list[list[int]] = []
    for op, pv in fuse_fold_iter(circuit, max_gate_size, max_diag_size, relabel_swaps):
        ops.append(op)
        prov.append(pv)
    return FoldedCircuit(ops, prov)


def fold_ops(circuit: Sequence[Gate], max_gate_size: int = 5, max_diag_size: int = 10,
             relabel_swaps: bool = True):
    """The fused ops one at a time, as the fuser closes each window: feeding
    them straight to ``run_circuit_sv`` overlaps host fusion with the GPU
    running the windows already emitted."""
    for op, _ in fuse_fold_iter(circuit, max_gate_size, max_diag_size, relabel_swaps):
        yield op


def fuse_fold_iter(circuit: Sequence[Gate], max_gate_size: int = 5, max_diag_size: int = 10,
                   relabel_swaps: bool = True):
    """Generator form of :func:`fuse_fold`: yields (op, provenance) pairs."""
    k = int(max_gate_size)
    if not 1 <= k <= 10 or not 1 <= max_diag_size <= 12:
        raise InvalidArgumentError("fusion sizes out of range")
    gates = list(circuit)
    phases = [_phase_poly(g) for g in gates]
    swaps = [relabel_swaps and _is_swap(g) for g in gates]
    remaining = list(range(len(gates)))

    qsets = [frozenset(g.qubits) for g in gates]  # computed once: the scan below revisits gates

    def qset(i):
        return qsets[i]

    while True:
        g0 = next((i for i in remaining if phases[i] is None), None)
        if g0 is None:
            break
        standalone = swaps[g0] or len(qset(g0)) > k
        W = set(qset(g0))                 # qubits owned by the window (g0 reserved up front)
        acted: set[int] = set()           # qubits a non-diagonal member already acted on
        members: list[int] = []           # matrix gates + internal phases, circuit order
        pre: list[int] = []               # phase gates applied before the window matrix
        left_nd: set[int] = set()         # qubits of left-behind matrix gates
        pending: list[tuple[int, bool]] = []  # left-behind phases (index, movable)
        taken: set[int] = set()

        fixed_q: set[int] = set()         # qubits of non-movable pending phases

        def absorb_pending(qs):
            """Movable pending phases touching qubits that join W become
            pre-phases (they precede every member acting on those qubits)."""
            if not any(mov for _, mov in pending):
                return
            keep = []
            for pi, mov in pending:
                if mov and not qsets[pi].isdisjoint(qs):
                    pre.append(pi)
                    taken.add(pi)
                else:
                    keep.append((pi, mov))
            pending[:] = keep

        def blocked_by_pending(qs) -> bool:
            return not fixed_q.isdisjoint(qs)

        for i in remaining:
            qs = qset(i)
            if phases[i] is not None:
                if standalone:
                    # phases before g0 on its qubits must be applied first
                    if i < g0 and qs & W:
                        pre.append(i)
                        taken.add(i)
                    continue
                if qs & left_nd:
                    pending.append((i, False))
                    fixed_q |= qs
                elif not (qs & acted):
                    if qs & W:
                        pre.append(i)          # precedes every member on its qubits
                        taken.add(i)
                    else:
                        pending.append((i, True))
                elif qs <= W:
                    members.append(i)          # internal, in circuit order
                    taken.add(i)
                else:
                    new = qs - W
                    if len(W | qs) <= k and not (new & left_nd) and not blocked_by_pending(new):
                        W |= new
                        absorb_pending(new)
                        members.append(i)
                        taken.add(i)
                    else:
                        pending.append((i, False))
                        fixed_q |= qs
                continue
            # matrix gate
            if i == g0:
                members.append(i)
                taken.add(i)
                acted |= qs
                absorb_pending(qs)
                if standalone:
                    break
                continue
            if (standalone or (qs & left_nd) or swaps[i] or len(W | qs) > k
                    or blocked_by_pending(qs)):
                left_nd |= qs
                continue
            new = qs - W
            W |= qs
            absorb_pending(qs)
            members.append(i)
            taken.add(i)
            acted |= qs
        remaining = [i for i in remaining if i not in taken]
        if standalone:
            if pre:
                yield _diag_window([gates[i] for i in pre], None), sorted(pre)
            g = gates[g0]
            yield (QubitSwap(*g.targets) if swaps[g0] else g), [g0]
            continue
        # movable single-qubit phases on outside qubits ride along as outside terms
        for pi, mov in pending:
            if mov and len(qset(pi)) == 1:
                pre.append(pi)
                taken.add(pi)
        remaining = [i for i in remaining if i not in taken]
        yield _emit_window(gates, phases, members, pre, W), sorted(members + pre)
    # leftover phase gates: commute with everything after them -> diagonal windows
    if remaining:
        for chunk in _pack_diagonals(remaining, gates, max_diag_size):
            yield _fused_diagonal([gates[i] for i in chunk], sorted({q for i in chunk for q in gates[i].qubits})), chunk


def _diag_window(gs, phs):
    return _fused_diagonal(gs, sorted({q for g in gs for q in g.qubits}))


def _pack_diagonals(idx: list[int], gates, limit: int) -> list[list[int]]:
    out: list[list[int]] = []
    cur: list[int] = []
    cq: set[int] = set()
    for i in idx:
        qs = set(gates[i].qubits)
        if cur and len(cq | qs) > limit:
            out.append(cur)
            cur, cq = [], set()
        cur.append(i)
        cq |= qs
    if cur:
        out.append(cur)
    return out


def _emit_window(gates, phases, members: list[int], pre: list[int], W: set[int]):
    union = sorted(W)
    # pre-phase terms: cross (a in W, b outside) and terms that ended up inside
    inner_pre = np.ones(1 << len(union), dtype=np.complex128)
    cross: dict[tuple[int, int], float] = {}
    outside: dict[int, float] = {}
    pos = {q: i for i, q in enumerate(union)}
    cols = np.arange(1 << len(union))
    const = 0.0
    for i in pre:
        ph = phases[i]
        const += ph.const
        for q, t in ph.lin.items():
            if q in pos:
                inner_pre *= np.where((cols >> pos[q]) & 1, cmath.exp(1j * t), 1.0)
            else:
                outside[q] = outside.get(q, 0.0) + t
        if len(ph.qubits) == 2 and ph.quad != 0.0:
            a, b = ph.qubits
            if a in pos and b in pos:
                inner_pre *= np.where(((cols >> pos[a]) & 1) & ((cols >> pos[b]) & 1), cmath.exp(1j * ph.quad), 1.0)
            else:
                ta, ob = (a, b) if a in pos else (b, a)
                cross[(ta, ob)] = cross.get((ta, ob), 0.0) + ph.quad
    prod = np.diag(inner_pre * cmath.exp(1j * const))
    for i in members:
        ph = phases[i]
        if ph is not None:  # internal phase: scale the rows (no 2^m x 2^m product)
            ang = np.full(cols.size, ph.const)
            for q, t in ph.lin.items():
                ang += t * ((cols >> pos[q]) & 1)
            if len(ph.qubits) == 2 and ph.quad != 0.0:
                a, b = ph.qubits
                ang += ph.quad * (((cols >> pos[a]) & 1) & ((cols >> pos[b]) & 1))
            prod *= np.exp(1j * ang)[:, None]
            continue
        prod = expand_gate(gates[i], union) @ prod
    if not cross and not outside:
        return DenseGate(prod, tuple(union), unitary=False)
    return PhasedDenseGate(prod, tuple(union), [(a, b, t) for (a, b), t in cross.items()],
                           [(b, t) for b, t in outside.items()])
