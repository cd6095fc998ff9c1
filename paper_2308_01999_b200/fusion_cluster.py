"""Cluster-merging gate fusion (opt-in): several fused
windows open at once, one per group of qubits, instead of the reference's
single scan window (fusion.py:124-179) or the fold fuser's one-window-at-a-
time scan (fusion_fold.py).

Every qubit belongs to at most one OPEN cluster.  A gate on qubits Q merges
the clusters that own Q (and Q itself) into one cluster when the union has
at most k qubits.  Otherwise touched clusters are closed — the one with the
most qubits first, it is the fullest and least able to grow — until the
union fits; a closed cluster becomes one fused dense gate (the time-ordered
product of its gates, fusion.fused_matrix).  Clusters are emitted in the
order they close, the still-open ones at the end.  Correctness of that order:
a qubit's gates fall into consecutive runs, one per cluster that owned it,
and a qubit joins a new cluster only after its previous cluster closed, so
per qubit the emitted order equals circuit order; clusters emitted "out of
circuit order" own disjoint qubits and commute.

On layered circuits of parallel 2-qubit gates this keeps the windows of one
layer open into the next: quantum volume depth 30 at n = 33 fuses into 134
windows at k = 5 (reference / fold fuser: 152) and QV-34 into 188 at k = 4
(232); a post-pass then merges windows that can be brought next to each
other by commuting past disjoint windows.  :func:`fuse_auto` returns
whichever of this and the fold fuser makes fewer data passes (QFT-like
circuits keep the fold fuser's phase folding: 7 passes for QFT-33).
"""

from __future__ import annotations

from collections.abc import Sequence

from .core import InvalidArgumentError
from .fusion import fused_matrix
from .fusion_fold import FoldedCircuit, fuse_fold
from .gates import Gate

__all__ = ["fuse_cluster", "fuse_auto"]


def fuse_cluster(circuit: Sequence[Gate], max_gate_size: int = 5) -> FoldedCircuit:
    """Fuse `circuit` into dense windows of <= max_gate_size qubits by
    cluster merging.  Gates wider than the limit pass through unchanged (as
    in the reference fuser, fusion.py:137-139) after closing the clusters
    they touch."""
    k = int(max_gate_size)
    if not 1 <= k <= 10:
        raise InvalidArgumentError("fusion size out of range")
    gates = list(circuit)
    owner: dict[int, int] = {}             # qubit -> open cluster id
    members: dict[int, list[int]] = {}     # cluster id -> gate indices (circuit order)
    qubits: dict[int, set[int]] = {}       # cluster id -> qubits
    order: list[int] = []                  # open cluster ids in creation order
    nxt = 0

    wins: list[tuple[list[int], set[int], bool]] = []  # (gate indices, qubits, mergeable) in emission order

    def close(cid: int) -> None:
        idx = members.pop(cid)
        qs = qubits.pop(cid)
        for q in qs:
            del owner[q]
        order.remove(cid)
        wins.append((idx, qs, True))

    for i, g in enumerate(gates):
        qs = set(g.qubits)
        cids = {owner[q] for q in qs if q in owner}
        if len(qs) > k:  # oversized: applied on its own after everything it touches
            for c in sorted(cids, key=order.index):
                close(c)
            wins.append(([i], qs, False))
            continue
        union = set(qs)
        for c in cids:
            union |= qubits[c]
        while len(union) > k:
            c = max(cids, key=lambda c: (len(qubits[c]), -order.index(c)))
            close(c)
            cids.discard(c)
            union = set(qs)
            for c2 in cids:
                union |= qubits[c2]
        merged = sorted((gi for c in cids for gi in members[c]))
        for c in cids:
            del members[c]
            del qubits[c]
            order.remove(c)
        cid = nxt
        nxt += 1
        members[cid] = merged + [i]
        qubits[cid] = union
        order.append(cid)
        for q in union:
            owner[q] = cid
    for c in list(order):
        close(c)
    wins = _merge_windows(wins, k)
    ops: list = []
    prov: list[list[int]] = []
    for idx, qs, _ in wins:
        if len(idx) == 1 and len(gates[idx[0]].qubits) == len(qs):
            ops.append(gates[idx[0]])       # a lone gate stays itself (diagonals keep their kind)
        else:
            ops.append(fused_matrix([gates[i] for i in idx], sorted(qs)))
        prov.append(idx)
    return FoldedCircuit(ops, prov)


def _merge_windows(wins, k: int):
    """Post-pass: window i merges into a later window j when their union has
    <= k qubits and either i commutes forward past every window in between
    (disjoint qubits) or j commutes backward past them — the merged window
    applies i's gates, then j's.  Repeated until nothing merges (QV-33 k=5:
    134 -> 130 windows, QV-34 k=4: 188 -> 181)."""
    wins = [(list(a), set(b), m) for a, b, m in wins]
    changed = True
    while changed:
        changed = False
        i = 0
        while i < len(wins):
            gi, qi, mi = wins[i]
            merged = False
            if mi:
                for j in range(i + 1, len(wins)):
                    gj, qj, mj = wins[j]
                    if mj and len(qi | qj) <= k:
                        between = wins[i + 1:j]
                        if all(w[1].isdisjoint(qi) for w in between):
                            wins[j] = (gi + gj, qi | qj, True)   # i moves forward to j
                            del wins[i]
                            merged = True
                            break
                        if all(w[1].isdisjoint(qj) for w in between):
                            wins[i] = (gi + gj, qi | qj, True)   # j moves back to i
                            del wins[j]
                            merged = True
                            break
            if merged:
                changed = True
            else:
                i += 1
    return wins


def fuse_auto(circuit: Sequence[Gate], max_gate_size: int = 5) -> FoldedCircuit:
    """The fold fuser or the cluster fuser, whichever makes fewer data passes
    over the state (ties: the fold fuser)."""
    gates = list(circuit)
    fold = fuse_fold(gates, max_gate_size)
    clus = fuse_cluster(gates, max_gate_size)
    return clus if clus.data_passes < fold.data_passes else fold
