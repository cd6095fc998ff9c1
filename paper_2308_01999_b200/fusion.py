"""Host gate fusion (mirror of ``duetsim.fusion``,
/root/reference/pkg/src/duetsim/fusion.py:1-179).

Greedy windowed pass, reference semantics (pinned by the reference's
test_fusion goldens — fused counts, provenance, idempotence):

* gates are visited in circuit order; a gate's *anchor* is the latest window
  that touched any of its qubits;
* a diagonal gate whose qubits all sit inside a (non-oversized) dense anchor
  window is absorbed into it;
* otherwise the gate joins the first window at or after the anchor of its own
  kind (dense / diagonal) whose qubit union stays within the size limit;
* otherwise it opens a new window; gates larger than the limit get a window
  of their own and pass through unchanged (same object).

Windows become one dense matrix (product of the members expanded onto the
sorted qubit union, controls in projector form) or one diagonal
PermutationGate.  The products are computed in complex128 on the host.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from .core import InvalidArgumentError
from .gates import DenseGate, Gate, PermutationGate

_MAX_FUSED_QUBITS = 10  # fusion.py:22


@dataclass
class FusionConfig:
    max_fused_gate_size: int = 4
    max_fused_diagonal_gate_size: int = 6

    def __post_init__(self):
        if min(self.max_fused_gate_size, self.max_fused_diagonal_gate_size) < 1:
            raise InvalidArgumentError("fusion sizes must be >= 1")


@dataclass
class FusedCircuit:
    gates: list[Gate]
    provenance: list[list[int]]

    def __len__(self) -> int:
        return len(self.gates)


@dataclass
class _Window:
    kind: str
    qubits: set[int]
    members: list[int] = field(default_factory=list)
    oversized: bool = False


def _kind(g: Gate) -> str:
    return "diag" if isinstance(g, PermutationGate) and g.is_diagonal else "dense"


def _bit_positions(union: Sequence[int], qubits: Sequence[int]) -> list[int]:
    where = {q: i for i, q in enumerate(union)}
    missing = [q for q in qubits if q not in where]
    if missing:
        raise InvalidArgumentError(f"gate qubit {missing[0]} not in union targets {list(union)}")
    return [where[q] for q in qubits]


def expand_gate(g: Gate, union_targets: Sequence[int]) -> np.ndarray:
    """2^m x 2^m matrix of ``g`` on the qubits ``union_targets`` (bit m of the
    expanded index is union_targets[m]); columns whose controls are not
    satisfied are identity (fusion.py:58-94)."""
    union = list(union_targets)
    m = len(union)
    if m > _MAX_FUSED_QUBITS:
        raise InvalidArgumentError(f"fused matrix over {m} qubits exceeds limit {_MAX_FUSED_QUBITS}")
    tpos = _bit_positions(union, g.targets)
    cpos = _bit_positions(union, [q for q, _ in g.controls])
    mat = g.matrix if isinstance(g, DenseGate) else g.to_matrix()
    dim = 1 << m
    col = np.arange(dim)
    ok = np.ones(dim, dtype=bool)
    for pos, (_, val) in zip(cpos, g.controls):
        ok &= ((col >> pos) & 1) == val
    out = np.zeros((dim, dim), dtype=np.complex128)
    idle = col[~ok]
    out[idle, idle] = 1.0
    act = col[ok]
    tmask = 0
    j_in = np.zeros(act.size, dtype=np.int64)
    for bit, pos in enumerate(tpos):
        j_in |= ((act >> pos) & 1) << bit
        tmask |= 1 << pos
    rest = act & ~tmask
    for j_out in range(1 << len(tpos)):
        row = rest.copy()
        for bit, pos in enumerate(tpos):
            if (j_out >> bit) & 1:
                row |= 1 << pos
        out[row, act] = mat[j_out, j_in]
    return out


def fused_matrix(gates: Sequence[Gate], union_targets: Sequence[int]) -> DenseGate:
    """Time-ordered product of ``gates`` on ``union_targets`` (fusion.py:97-103)."""
    prod = np.eye(1 << len(union_targets), dtype=np.complex128)
    for g in gates:
        prod = expand_gate(g, union_targets) @ prod
    unit = all(g.unitary for g in gates if isinstance(g, DenseGate))
    return DenseGate(prod, tuple(union_targets), unitary=unit)


def _fused_diagonal(gates: Sequence[PermutationGate], union_targets: Sequence[int]) -> PermutationGate:
    """Entry-wise product of diagonal gates on the union (fusion.py:106-121)."""
    union = list(union_targets)
    dim = 1 << len(union)
    col = np.arange(dim)
    diag = np.ones(dim, dtype=np.complex128)
    for g in gates:
        cpos = _bit_positions(union, [q for q, _ in g.controls])
        ok = np.ones(dim, dtype=bool)
        for pos, (_, val) in zip(cpos, g.controls):
            ok &= ((col >> pos) & 1) == val
        j = np.zeros(dim, dtype=np.int64)
        for bit, pos in enumerate(_bit_positions(union, g.targets)):
            j |= ((col >> pos) & 1) << bit
        diag *= np.where(ok, g.diagonal[j], 1.0)
    return PermutationGate(np.arange(dim), diag, tuple(union))


def _plan_windows(circuit: Sequence[Gate], cfg: FusionConfig) -> list[_Window]:
    windows: list[_Window] = []
    last: dict[int, int] = {}
    for idx, g in enumerate(circuit):
        qs = set(g.qubits)
        kind = _kind(g)
        limit = cfg.max_fused_diagonal_gate_size if kind == "diag" else cfg.max_fused_gate_size
        anchor = max((last.get(q, -1) for q in qs), default=-1)
        target: int | None = None
        if len(qs) > limit:
            windows.append(_Window(kind, set(qs), [idx], oversized=True))
            target = len(windows) - 1
        else:
            if kind == "diag" and anchor >= 0:
                a = windows[anchor]
                if a.kind == "dense" and not a.oversized and qs <= a.qubits:
                    target = anchor
            if target is None:
                for i in range(max(anchor, 0), len(windows)):
                    w = windows[i]
                    if not w.oversized and w.kind == kind and len(w.qubits | qs) <= limit:
                        target = i
                        break
            if target is None:
                windows.append(_Window(kind, set(qs), [idx]))
                target = len(windows) - 1
            else:
                windows[target].qubits |= qs
                windows[target].members.append(idx)
        for q in qs:
            last[q] = target
    return windows


def fuse(circuit: Sequence[Gate], cfg: FusionConfig | None = None) -> FusedCircuit:
    """Compile a gate list into fused dense windows and diagonal runs
    (fusion.py:124-179)."""
    cfg = cfg or FusionConfig()
    out: list[Gate] = []
    prov: list[list[int]] = []
    for w in _plan_windows(circuit, cfg):
        if len(w.members) == 1:
            out.append(circuit[w.members[0]])
        else:
            union = sorted(w.qubits)
            members = [circuit[i] for i in w.members]
            out.append(_fused_diagonal(members, union) if w.kind == "diag" else fused_matrix(members, union))
        prov.append(list(w.members))
    return FusedCircuit(out, prov)
