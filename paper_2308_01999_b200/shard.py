"""One host process driving P = 2^g GPUs: a 2^n state vector sharded by its
top g index bits, PyTorch-free (the reference's SegmentedStateVector with one
segment per device, distsim.py:69-277, as SURVEY.md §8(b) lays out the C ABI:
one host thread, every device reached through libdsv).

* Local gates (all targets local) are queued on every segment's stream; the
  calls return at once, so all P devices run the gate concurrently.  A
  segment whose global control bits disagree skips the gate
  (distsim.py:232-244).
* A global target is relocated first with the reference's victim choice
  (furthest next use as a target, distsim.py:202-221), ties broken toward the
  HIGHEST local bit so the exchange moves long contiguous runs.  All (global,
  local) pairs of one reorder are executed together (plan.exchange_rounds):
  2^q - 1 rounds of pairwise exchanges, each a single in-place pass of the
  masked exchange kernel over peer memory (NVLink / NVSwitch), split half
  and half between the two partner GPUs and stream-ordered with events — no
  host synchronisation, no staging buffer, no NCCL on amplitude data.
* Reductions (norm, marginals, Pauli expectations) run on every device at
  once (dsv_group_*) and the P partial results are combined on the host in
  segment order (deterministic).

``devices`` may repeat a device id: P segments on one GPU exercise the same
host protocol and kernels (the P-invariance tests on a 1-GPU box).
"""

from __future__ import annotations

import math
from collections.abc import Sequence

import numpy as np

from . import _native as N
from .core import InvalidArgumentError, check_swap_pairs
from .gates import Gate, PauliString, PermutationGate
from .plan import (TransferStats, decompose_swap, exchange_rounds, initial_placement, localize_phased, relabel,
                   relocation_pairs, segment_selected, split_controls, swap_transfer)

__all__ = ["ShardedStateVector", "batched_exchange"]


def _group(segs, name: str, *args):
    """Per-segment reduction over the group: libdsv's dsv_group_* (all
    devices at once) or the segment class's own (CPU test doubles)."""
    fn = getattr(type(segs[0]), "group_" + name, None)
    if fn is None:
        fn = getattr(N, "group_" + name)
    return fn(segs, *args)


def batched_exchange(segs: Sequence[N.NativeState], global_local) -> None:
    """Execute the (global, local) part of an index-bit swap over segments
    `segs` (list index = global-bit value) as 2^q - 1 rounds of pairwise
    masked exchanges, each split over both partners' devices."""
    for _, s, t, lbits, pat_s, pat_t in exchange_rounds(global_local, len(segs)):
        segs[s].exchange_pair(segs[t], lbits, pat_s, pat_t)


def relabel_segments(segs: list, global_global, nseg: int) -> list:
    """(global, global) pairs move whole segments: relabel, no data moves."""
    for j1, j2 in global_global:
        out = list(segs)
        for s in range(nseg):
            if ((s >> j1) ^ (s >> j2)) & 1:
                out[s] = segs[s ^ ((1 << j1) | (1 << j2))]
        segs = out
    return segs


class ShardedStateVector:
    """2^n amplitudes over len(devices) = 2^g segments, one per device."""

    def __init__(self, num_qubits: int, devices: Sequence[int], dtype=np.complex64, segment_factory=None):
        devices = [int(d) for d in devices]
        P = len(devices)
        g = int(round(math.log2(P))) if P > 0 else -1
        if P < 1 or (1 << g) != P:
            raise InvalidArgumentError(f"{P} devices: the segment count must be a power of two")
        if not 0 <= g < num_qubits:
            raise InvalidArgumentError("need fewer global bits than qubits")
        self.num_qubits = num_qubits
        self.global_bits = g
        self.local_bits = num_qubits - g
        self.dtype = np.dtype(dtype)
        self.devices = devices
        make = segment_factory or N.NativeState
        self.segs: list[N.NativeState] = []
        for s, d in enumerate(devices):
            st = make(self.local_bits, self.dtype, d)
            if s:
                st.set_zero()
            self.segs.append(st)
        self.qubit_map = list(range(num_qubits))
        self.stats = TransferStats()
        self._basis0 = True

    # -- plumbing --------------------------------------------------------------------
    @property
    def num_segments(self) -> int:
        return len(self.segs)

    def sync(self) -> None:
        for st in self.segs:
            st.sync()

    def close(self) -> None:
        self.sync()
        for st in self.segs:
            st.close()
        self.segs = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def reset(self) -> None:
        """|0...0> with the identity qubit map."""
        for s, st in enumerate(self.segs):
            if s == 0:
                st.set_basis(0)
            else:
                st.set_zero()
        self.qubit_map = list(range(self.num_qubits))
        self._basis0 = True

    # -- layout --------------------------------------------------------------------------
    def distributed_index_bit_swap(self, pairs: Sequence[tuple[int, int]]) -> None:
        """swap_index_bits of the whole vector (distsim.py:153-198): local
        pairs on every segment, (global, local) pairs as batched P2P rounds,
        (global, global) pairs as a segment relabel; qubit_map relabelled."""
        check_swap_pairs(pairs)
        n = self.num_qubits
        for a, b in pairs:
            if a >= n or b >= n:
                raise InvalidArgumentError(f"bit pair ({a}, {b}) exceeds {n} bits")
        pairs = [(int(a), int(b)) for a, b in pairs]
        dec = decompose_swap(pairs, self.local_bits)
        if dec.local_pairs:
            for st in self.segs:
                st.swap_bits(dec.local_pairs)
        if dec.global_local:
            batched_exchange(self.segs, dec.global_local)
        if dec.global_global:
            self.segs = relabel_segments(self.segs, dec.global_global, len(self.segs))
        ex, moved, intra, inter = swap_transfer(pairs, self.local_bits, self.global_bits, len(self.segs))
        if ex:
            self.stats.num_reorders += 1
            self.stats.num_messages += 2 * ex
            self.stats.amplitudes_moved += moved
            self.stats.amplitudes_moved_intra_worker += intra
            self.stats.amplitudes_moved_inter_worker += inter
        self.qubit_map = relabel(self.qubit_map, pairs)

    def _relocate(self, target_bits, upcoming) -> None:
        pairs = relocation_pairs(self.qubit_map, self.local_bits, target_bits, upcoming, prefer_high=True)
        if pairs:
            self.distributed_index_bit_swap(pairs)

    # -- gates ---------------------------------------------------------------------------------
    def apply(self, g: Gate, upcoming=()) -> None:
        """apply_gate_distributed (distsim.py:223-259) for one gate or fold-
        fuser op, queued on every selected segment."""
        from .fusion_fold import PhasedDenseGate, QubitSwap

        self._basis0 = False
        if isinstance(g, QubitSwap):  # relabel only
            self.qubit_map[g.a], self.qubit_map[g.b] = self.qubit_map[g.b], self.qubit_map[g.a]
            return
        if len(g.targets) > self.local_bits:
            raise InvalidArgumentError(f"gate arity {len(g.targets)} exceeds local capacity {self.local_bits}")
        for q in g.qubits:
            if not 0 <= q < self.num_qubits:
                raise InvalidArgumentError(f"qubit {q} out of range")
        self._relocate([self.qubit_map[q] for q in g.targets], upcoming)
        if isinstance(g, PhasedDenseGate):
            for s, st in enumerate(self.segs):
                m, tb, cross, outside = localize_phased(g, self.qubit_map, self.local_bits, s, self.dtype)
                st.apply_matrix_phased(m, tb, cross, outside)
            return
        tbits = [self.qubit_map[q] for q in g.targets]
        loc, glob = split_controls(self.qubit_map, self.local_bits, g.controls)
        if isinstance(g, PermutationGate):
            diag = np.asarray(g.diagonal, dtype=self.dtype)
            for s, st in enumerate(self.segs):
                if segment_selected(s, glob):
                    st.apply_genperm(g.permutation, diag, tbits, loc)
        else:
            mat = np.asarray(g.matrix, dtype=self.dtype)
            for s, st in enumerate(self.segs):
                if segment_selected(s, glob):
                    st.apply_matrix(mat, tbits, loc)

    def run(self, gates) -> None:
        """Run a gate list (distsim.py:261-264); from |0...0> the qubit map
        is first chosen so the global qubits are the ones targeted last."""
        gates = list(gates)
        if self._basis0 and self.global_bits > 0:
            self.qubit_map = initial_placement(gates, self.num_qubits, self.local_bits)
        for i, g in enumerate(gates):
            self.apply(g, gates[i + 1:])

    # -- reductions --------------------------------------------------------------------------------
    def norm_squared(self) -> float:
        return float(sum(_group(self.segs, 'norm2')))

    def probabilities(self, qubits: Sequence[int]) -> np.ndarray:
        """Marginal probabilities over `qubits` (statevec.py:209-213 order:
        entry o has bit j = value of qubits[j])."""
        qubits = [int(q) for q in qubits]
        if len(set(qubits)) != len(qubits):
            raise InvalidArgumentError("qubits must be distinct")
        for q in qubits:
            if not 0 <= q < self.num_qubits:
                raise InvalidArgumentError(f"qubit {q} out of range")
        bits = [self.qubit_map[q] for q in qubits]
        loc_pos = [j for j, b in enumerate(bits) if b < self.local_bits]
        if loc_pos:
            local = _group(self.segs, 'marginal', [bits[j] for j in loc_pos])
        else:
            local = _group(self.segs, 'norm2')[:, None]
        out = np.zeros(1 << len(bits))
        o_loc = np.arange(local.shape[1])
        spread = np.zeros_like(o_loc)
        for t, j in enumerate(loc_pos):
            spread |= ((o_loc >> t) & 1) << j
        for s in range(len(self.segs)):
            gv = 0
            for j, b in enumerate(bits):
                if b >= self.local_bits and (s >> (b - self.local_bits)) & 1:
                    gv |= 1 << j
            np.add.at(out, gv | spread, local[s])
        return out

    def expectation(self, paulis: Sequence[PauliString]) -> complex:
        """sum_P coef_P <psi|P|psi>: X/Y factors on global qubits are
        relocated first (logical state unchanged), Z factors on global qubits
        become a per-segment sign."""
        total = 0.0 + 0.0j
        for pauli in paulis:
            if not isinstance(pauli, PauliString):
                raise InvalidArgumentError("sharded expectation takes a list of PauliString")
            flip = [self.qubit_map[q] for q, p in pauli.factors if p in "XY"]
            self._relocate(flip, [])
            local, gz = [], []
            for q, p in pauli.factors:
                bit = self.qubit_map[q]
                if bit < self.local_bits:
                    local.append((bit, p))
                elif p == "Z":
                    gz.append(bit - self.local_bits)
            parts = _group(self.segs, 'expect_pauli', local)
            acc = 0.0 + 0.0j
            for s, v in enumerate(parts):
                acc += -v if sum((s >> j) & 1 for j in gz) & 1 else v
            total += pauli.coefficient * acc
        return total

    # -- verification / instrumentation -------------------------------------------------------
    def gather_logical(self) -> np.ndarray:
        """Logical-order state on the host (tests only; O(2^n) memory)."""
        phys = np.concatenate([st.download() for st in self.segs])
        n = self.num_qubits
        idx = np.arange(1 << n, dtype=np.int64)
        src = np.zeros_like(idx)
        for q, bit in enumerate(self.qubit_map):
            src |= ((idx >> q) & 1) << bit
        return phys[src]

    def physical_segments(self) -> list[np.ndarray]:
        return [st.download() for st in self.segs]

    def prof(self, on: bool) -> None:
        for st in self.segs:
            st.prof_reset()
            st.prof_enable(on)

    def prof_read(self) -> list[dict]:
        return [st.prof_read() for st in self.segs]

    def event_record(self, slot: int) -> None:
        for st in self.segs:
            st.event_record(slot)

    def event_elapsed_max(self, a: int, b: int) -> float:
        """Device time between two recorded slots, max over segments (the
        exchanges join the streams, so each segment's span covers the work it
        waited for)."""
        return max(st.event_elapsed(a, b) for st in self.segs)
