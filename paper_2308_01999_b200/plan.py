"""Host-side planning for sharded state vectors (pure Python, no device).

Shared by the single-process :class:`~.distsim.SegmentedStateVector` and the
one-process-per-GPU :mod:`.multigpu` layer.  It restates the reference's
scheduling decisions analytically (distsim.py:122-221) instead of
materialising per-amplitude index arrays (2^36 entries at 36 qubits):

* which (global, local) index-bit swaps make a gate's targets local, with the
  reference's victim rule (furthest next use as a target; ties -> lowest bit);
* how a multi-pair index-bit swap decomposes into local permutations,
  pairwise half-segment exchanges and whole-segment relabels;
* the reference's TransferStats counters for that swap, in closed form.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass

from .core import InvalidArgumentError


@dataclass
class TransferStats:
    """Exchange counters (reference distsim.py:51-66)."""

    num_reorders: int = 0
    num_messages: int = 0
    amplitudes_moved: int = 0
    amplitudes_moved_intra_worker: int = 0
    amplitudes_moved_inter_worker: int = 0

    def as_dict(self) -> dict:
        return {
            "num_reorders": self.num_reorders,
            "num_messages": self.num_messages,
            "amplitudes_moved": self.amplitudes_moved,
            "amplitudes_moved_intra_worker": self.amplitudes_moved_intra_worker,
            "amplitudes_moved_inter_worker": self.amplitudes_moved_inter_worker,
        }


@dataclass
class SwapDecomposition:
    local_pairs: list[tuple[int, int]]            # both bits local
    global_local: list[tuple[int, int]]           # (segment bit j, local bit l)
    global_global: list[tuple[int, int]]          # (segment bit j1, segment bit j2)


def decompose_swap(pairs: Sequence[tuple[int, int]], nloc: int) -> SwapDecomposition:
    """Split disjoint bit pairs by locality.  Applying the three groups one
    after the other realises the same index permutation as the combined swap
    because disjoint bit transpositions commute."""
    loc, gl, gg = [], [], []
    for a, b in pairs:
        if a == b:
            continue
        ga, gb = a >= nloc, b >= nloc
        if not ga and not gb:
            loc.append((a, b))
        elif ga and gb:
            gg.append((a - nloc, b - nloc))
        else:
            gbit, lbit = (a, b) if ga else (b, a)
            gl.append((gbit - nloc, lbit))
    return SwapDecomposition(loc, gl, gg)


def swap_transfer(pairs: Sequence[tuple[int, int]], nloc: int, global_bits: int, workers: int):
    """Closed-form TransferStats increments of the reference's plan for this
    swap (distsim.py:185-194): returns (exchanges, moved, intra, inter).

    For segment s, a (global, local) pair can always move amplitudes to the
    segment with that global bit flipped; a (global, global) pair moves
    amplitudes only if s's two bits differ.  Each exchange between two
    segments carries 2 * seg_len * 2^-#GL amplitudes in total."""
    d = decompose_swap(pairs, nloc)
    nseg = 1 << global_bits
    seg_len = 1 << nloc
    gl_mask = 0
    for j, _ in d.global_local:
        gl_mask |= 1 << j
    per_exchange = 2 * seg_len >> len(d.global_local)
    exchanges = moved = intra = inter = 0
    for s in range(nseg):
        gg_flip = 0
        for j1, j2 in d.global_global:
            if ((s >> j1) ^ (s >> j2)) & 1:
                gg_flip |= (1 << j1) | (1 << j2)
        # destinations: GG swaps applied to s, GL bits free (they take the
        # value of the paired local bit, amplitude by amplitude)
        dests = []
        sub = gl_mask
        while True:
            dests.append(s ^ gg_flip ^ sub)
            if sub == 0:
                break
            sub = (sub - 1) & gl_mask
        for t in dests:
            if t > s:
                exchanges += 1
                moved += per_exchange
                if s % workers == t % workers:
                    intra += per_exchange
                else:
                    inter += per_exchange
    return exchanges, moved, intra, inter


def relabel(qubit_map: list[int], pairs: Sequence[tuple[int, int]]) -> list[int]:
    swapped = {}
    for a, b in pairs:
        swapped[a], swapped[b] = b, a
    return [swapped.get(bit, bit) for bit in qubit_map]


def relocation_pairs(qubit_map: Sequence[int], nloc: int, target_bits: Sequence[int],
                     upcoming, prefer_high: bool = False) -> list[tuple[int, int]]:
    """(global, local) swaps that make every target bit local
    (distsim.py:202-221): victims are local non-target bits whose qubit is
    next used as a target furthest in the future (never: first); ties go to
    the lowest bit — the reference's rule, which the drop-in
    SegmentedStateVector keeps so its qubit_map matches.  The sharded engines
    pass prefer_high=True: ties go to the HIGHEST local bit, so the exchange
    moves long contiguous runs instead of every other amplitude."""
    need = [b for b in target_bits if b >= nloc]
    if not need:
        return []
    owner = {bit: q for q, bit in enumerate(qubit_map)}
    horizon = len(upcoming) + 1
    next_use: dict[int, int] = {}
    for dist, g in enumerate(upcoming):
        for q in getattr(g, "targets", ()):
            next_use.setdefault(q, dist)
    cands = [b for b in range(nloc) if b not in target_bits]
    if len(need) > len(cands):
        raise InvalidArgumentError("gate arity exceeds local capacity")
    cands.sort(key=lambda b: (-next_use.get(owner[b], horizon), -b if prefer_high else b))
    return [(gb, cands[i]) for i, gb in enumerate(need)]


def split_controls(qubit_map: Sequence[int], nloc: int, controls):
    """Local controls as (bit, value); global ones as (segment bit, value)."""
    loc, glob = [], []
    for q, v in controls:
        bit = qubit_map[q]
        if bit < nloc:
            loc.append((bit, int(v)))
        else:
            glob.append((bit - nloc, int(v)))
    return loc, glob


def segment_selected(s: int, global_controls) -> bool:
    return all(((s >> b) & 1) == v for b, v in global_controls)


def localize_phased(op, qubit_map: Sequence[int], nloc: int, seg: int, dtype):
    """Per-segment form of a fold-fuser PhasedDenseGate whose targets are
    local: phase terms on GLOBAL outside qubits are constants inside a segment,
    so a cross term t x_a x_b (b global) becomes a phase on the target columns
    with bit a set, and an outside term on a global qubit a scalar phase.
    Returns (matrix, target_bits, cross[(m, bit, t)], outside[(bit, t)])."""
    import cmath

    import numpy as np

    m = np.array(op.matrix, dtype=np.complex128, copy=True)
    pos = {q: i for i, q in enumerate(op.targets)}
    cols = np.arange(m.shape[1])
    cross, outside = [], []
    for a, b, t in op.cross:
        bit = qubit_map[b]
        if bit < nloc:
            cross.append((pos[a], bit, t))
        elif (seg >> (bit - nloc)) & 1:
            m[:, ((cols >> pos[a]) & 1) == 1] *= cmath.exp(1j * t)
    for b, t in op.outside:
        bit = qubit_map[b]
        if bit < nloc:
            outside.append((bit, t))
        elif (seg >> (bit - nloc)) & 1:
            m *= cmath.exp(1j * t)
    return m.astype(dtype), [qubit_map[q] for q in op.targets], cross, outside


def initial_placement(gates, n: int, nloc: int) -> list[int]:
    """Qubit map for a state that is still |0...0>: that state is invariant
    under any relabelling of index bits, so before the first gate the map is
    free.  Put on the global bits the qubits whose first use as a target comes
    last (never: first), so e.g. a QFT needs one global<->local reorder
    instead of two.  No data moves; only the map changes."""
    ng = n - nloc
    first: dict[int, int] = {}
    for i, g in enumerate(gates):
        for q in getattr(g, "targets", ()):
            first.setdefault(q, i)
    glob = [q for q in range(n) if q not in first][:ng]
    if len(glob) < ng:
        # the latest gate that first-targets enough qubits takes all the
        # remaining global slots: one reorder brings them in together
        need = ng - len(glob)
        for i in range(len(gates) - 1, -1, -1):
            fresh = [q for q in getattr(gates[i], "targets", ()) if first.get(q) == i and q not in glob]
            if len(fresh) >= need:
                glob += sorted(fresh)[:need]
                break
    if len(glob) < ng:  # fall back: qubits whose first use as a target comes last
        order = sorted((q for q in range(n) if q not in glob), key=lambda q: (-first.get(q, len(gates) + 1), -q))
        glob += order[: ng - len(glob)]
    loc = [q for q in range(n) if q not in glob]
    qmap = [0] * n
    for b, q in enumerate(loc):
        qmap[q] = b
    for j, q in enumerate(sorted(glob)):
        qmap[q] = nloc + j
    return qmap


def exchange_rounds(global_local: Sequence[tuple[int, int]], nseg: int):
    """Schedule of a batched (global, local) swap of q pairs (j_i, l_i) over
    nseg segments: round m (a nonzero q-bit mask) pairs every segment s with
    t = s ^ M(m), M flipping the global bits j_i selected by m — a perfect
    matching, so every segment works in every round.  Segment s sends t the
    amplitudes whose local bits l_i equal t's bits j_i and receives those of t
    whose l_i equal s's j_i:  a_s[off | pat(t)] <-> a_t[off | pat(s)].
    Each amplitude moves at most once: a q-bit swap moves (1 - 2^-q) of the
    vector in 2^q - 1 rounds instead of q/2 of it per pair done one by one.
    Yields (round, s, t, lbits, pat_s_side, pat_t_side) with s < t."""
    js = [j for j, _ in global_local]
    ls = [l for _, l in global_local]
    q = len(js)

    def pat(seg: int) -> int:
        return sum(((seg >> j) & 1) << l for j, l in zip(js, ls))

    for m in range(1, 1 << q):
        flip = sum(1 << js[i] for i in range(q) if (m >> i) & 1)
        for s in range(nseg):
            t = s ^ flip
            if s < t:
                yield m, s, t, ls, pat(t), pat(s)
