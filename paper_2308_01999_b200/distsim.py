"""Segmented state vector (drop-in for ``duetsim.distsim``,
/root/reference/pkg/src/duetsim/distsim.py).

The 2^n amplitudes are split into 2^g equal segments: index bits below n-g
are local, the top g bits select the segment.  Each segment is a libdsv
device segment (one HBM allocation, its own CUDA stream); segments are
spread round-robin over ``devices`` (default: one device).  Gates only run
on local bits; a global target is first swapped with a local "victim" bit.

The reference stages full segment copies and scatters with per-amplitude
index arrays (distsim.py:153-198).  Here a (global, local) swap is one
in-place pass of the masked exchange kernel per segment pair, all (global,
local) pairs of one swap batched into 2^q - 1 rounds (shard.batched_exchange;
peer access when the two segments sit on different GPUs, the work split
between both), local pairs use the in-place bit swap kernel, and (global, global) pairs relabel whole segments without
moving data.  TransferStats keeps the reference's accounting (closed form,
see plan.py).  For the one-process-per-GPU layer see multigpu.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import InvalidArgumentError, bit_permute_array, check_swap_pairs
from .gates import Gate, PauliString, PermutationGate
from .plan import (
    TransferStats,
    decompose_swap,
    localize_phased,
    relabel,
    relocation_pairs,
    segment_selected,
    split_controls,
    swap_transfer,
)
from .mirror import mirror_of
from .shard import batched_exchange, relabel_segments
from .statevec import StateVector

__all__ = ["Exchange", "ReorderPlan", "TransferStats", "SegmentedStateVector"]


@dataclass
class Exchange:
    """One two-party exchange of a reorder schedule (distsim.py:28-37)."""

    seg_a: int
    src_a: np.ndarray
    dst_b: np.ndarray
    seg_b: int
    src_b: np.ndarray
    dst_a: np.ndarray


@dataclass
class ReorderPlan:
    swaps: list[tuple[int, int]]
    exchanges: list[Exchange]
    local_perm: dict[int, tuple[np.ndarray, np.ndarray]]

    @property
    def amplitudes_moved(self) -> int:
        return sum(len(e.src_a) + len(e.src_b) for e in self.exchanges)


class _Mirrors(list):
    """The host view handed out by ``segments``: a list of NumPy arrays the
    caller may mutate in place; uploaded before the next device operation."""


class SegmentedStateVector:
    def __init__(self, num_qubits: int, global_bits: int, workers: int = 1, dtype=np.complex128,
                 devices=None):
        if not (0 < global_bits < num_qubits):
            raise InvalidArgumentError("need 0 < global_bits < num_qubits")
        if workers < 1:
            raise InvalidArgumentError("workers must be >= 1")
        self.num_qubits = num_qubits
        self.global_bits = global_bits
        self.local_bits = num_qubits - global_bits
        self.workers = workers
        self.dtype = np.dtype(dtype)
        devs = list(devices) if devices is not None else [N.default_device()]
        self._devs: list[N.NativeState] = []
        for s in range(1 << global_bits):
            st = N.NativeState(self.local_bits, self.dtype, devs[s % len(devs)])
            if s:
                st.set_zero()
            self._devs.append(st)
        self.qubit_map = list(range(num_qubits))
        self.stats = TransferStats()
        self._mirrors: _Mirrors | None = None
        self._mirror_valid = False
        self._host_dirty = False

    # -- plumbing -------------------------------------------------------------
    def close(self) -> None:
        for st in self._devs:
            st.sync()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def worker_of(self, segment: int) -> int:
        return segment % self.workers

    @property
    def segments(self) -> list[np.ndarray]:
        if not self._mirror_valid:
            if self._mirrors is None:
                self._mirrors = _Mirrors(np.empty(1 << self.local_bits, dtype=self.dtype) for _ in self._devs)
            for st, m in zip(self._devs, self._mirrors):
                st.download(m)
            self._mirror_valid = True
        # writes into a segment array flag the mirrors for upload (mirror.py);
        # reads alone never re-upload
        return _Mirrors(mirror_of(m, self.mark_host_dirty) for m in self._mirrors)

    def mark_host_dirty(self) -> None:
        if self._mirrors is not None and self._mirror_valid:
            self._host_dirty = True

    def _sync_in(self) -> None:
        if self._host_dirty and self._mirror_valid and self._mirrors is not None:
            for st, m in zip(self._devs, self._mirrors):
                st.upload(m)
        self._host_dirty = False

    def _mutated(self) -> None:
        self._mirror_valid = False
        self._host_dirty = False

    @property
    def native_segments(self) -> list[N.NativeState]:
        self._sync_in()
        return list(self._devs)

    # -- reordering -----------------------------------------------------------------
    def _check_pairs(self, pairs) -> list[tuple[int, int]]:
        check_swap_pairs(pairs)
        n = self.num_qubits
        for a, b in pairs:
            if a >= n or b >= n:
                raise InvalidArgumentError(f"bit pair ({a}, {b}) exceeds {n} bits")
        return [(int(a), int(b)) for a, b in pairs]

    def plan_index_bit_swap(self, pairs) -> ReorderPlan:
        """Explicit per-amplitude schedule (distsim.py:122-151), materialised
        on the host for inspection.  Execution never builds it."""
        pairs = self._check_pairs(pairs)
        nloc = self.local_bits
        if nloc > 24:
            raise InvalidArgumentError("explicit reorder plans are only materialised for <= 24 local bits")
        offs = np.arange(1 << nloc, dtype=np.int64)
        low = (1 << nloc) - 1
        moves: dict[tuple[int, int], tuple[np.ndarray, np.ndarray]] = {}
        local_perm: dict[int, tuple[np.ndarray, np.ndarray]] = {}
        for s in range(len(self._devs)):
            dest = bit_permute_array((s << nloc) | offs, pairs)
            dseg, doff = dest >> nloc, dest & low
            for t in np.unique(dseg):
                t = int(t)
                sel = dseg == t
                if t == s:
                    if np.any(doff[sel] != offs[sel]):
                        local_perm[s] = (offs[sel], doff[sel])
                else:
                    moves[(s, t)] = (offs[sel], doff[sel])
        exchanges = [
            Exchange(a, sa, db, b, *moves[(b, a)])
            for (a, b), (sa, db) in sorted(moves.items())
            if a < b
        ]
        return ReorderPlan(pairs, exchanges, local_perm)

    def distributed_index_bit_swap(self, pairs) -> None:
        """Swap index-bit pairs of the concatenated vector in place and update
        the qubit map (distsim.py:153-198)."""
        pairs = self._check_pairs(pairs)
        self._sync_in()
        dec = decompose_swap(pairs, self.local_bits)
        nseg = len(self._devs)
        if dec.local_pairs:
            for st in self._devs:
                st.swap_bits(dec.local_pairs)
        if dec.global_local:
            batched_exchange(self._devs, dec.global_local)
        if dec.global_global:
            self._devs = relabel_segments(self._devs, dec.global_global, nseg)
        self._mutated()
        ex, moved, intra, inter = swap_transfer(pairs, self.local_bits, self.global_bits, self.workers)
        if ex:
            self.stats.num_reorders += 1
            self.stats.num_messages += 2 * ex
            self.stats.amplitudes_moved += moved
            self.stats.amplitudes_moved_intra_worker += intra
            self.stats.amplitudes_moved_inter_worker += inter
        self.qubit_map = relabel(self.qubit_map, pairs)

    # -- gate application ----------------------------------------------------------------
    def _relocation_pairs(self, target_bits, upcoming) -> list[tuple[int, int]]:
        return relocation_pairs(self.qubit_map, self.local_bits, target_bits, upcoming)

    def apply_gate_distributed(self, g: Gate, upcoming=()) -> None:
        """distsim.py:223-259.  Gate data is cast to the state dtype
        (StateVector semantics, SURVEY §7.3 hard part 3).  Also accepts the
        fold fuser's ops (fusion_fold.py): QubitSwap relabels the qubit map,
        PhasedDenseGate runs per segment with global phase qubits folded in."""
        from .fusion_fold import PhasedDenseGate, QubitSwap

        if isinstance(g, QubitSwap):
            self.qubit_map[g.a], self.qubit_map[g.b] = self.qubit_map[g.b], self.qubit_map[g.a]
            return
        if isinstance(g, PhasedDenseGate):
            pairs = self._relocation_pairs([self.qubit_map[q] for q in g.targets], upcoming)
            if pairs:
                self.distributed_index_bit_swap(pairs)
            self._sync_in()
            for s, st in enumerate(self._devs):
                m, tb, cross, outside = localize_phased(g, self.qubit_map, self.local_bits, s, self.dtype)
                st.apply_matrix_phased(m, tb, cross, outside)
            self._mutated()
            return
        if len(g.targets) > self.local_bits:
            raise InvalidArgumentError(
                f"gate arity {len(g.targets)} exceeds local capacity {self.local_bits}"
            )
        for q in g.qubits:
            if not 0 <= q < self.num_qubits:
                raise InvalidArgumentError(f"qubit {q} out of range")
        pairs = self._relocation_pairs([self.qubit_map[q] for q in g.targets], upcoming)
        if pairs:
            self.distributed_index_bit_swap(pairs)
        self._sync_in()
        tbits = [self.qubit_map[q] for q in g.targets]
        loc, glob = split_controls(self.qubit_map, self.local_bits, g.controls)
        if isinstance(g, PermutationGate):
            diag = np.asarray(g.diagonal, dtype=self.dtype)
            for s, st in enumerate(self._devs):
                if segment_selected(s, glob):
                    st.apply_genperm(g.permutation, diag, tbits, loc)
        else:
            mat = np.asarray(g.matrix, dtype=self.dtype)
            for s, st in enumerate(self._devs):
                if segment_selected(s, glob):
                    st.apply_matrix(mat, tbits, loc)
        self._mutated()

    def run(self, gates) -> None:
        gates = list(gates)
        for i, g in enumerate(gates):
            self.apply_gate_distributed(g, upcoming=gates[i + 1:])

    def transfer_stats(self) -> TransferStats:
        return self.stats

    # -- reductions (extension: the reference has none; BASELINE config 5) ------------
    def norm_squared(self) -> float:
        self._sync_in()
        return float(sum(st.norm2() for st in self._devs))

    def expectation(self, paulis) -> complex:
        """sum_P coef_P <psi|P|psi> over all segments.  X/Y factors on global
        qubits are relocated first (logical state unchanged); Z factors on
        global qubits become a per-segment sign."""
        total = 0.0 + 0.0j
        for pauli in paulis:
            if not isinstance(pauli, PauliString):
                raise InvalidArgumentError("segmented expectation takes a list of PauliString")
            flip = [self.qubit_map[q] for q, p in pauli.factors if p in "XY"]
            pairs = relocation_pairs(self.qubit_map, self.local_bits, flip, [])
            if pairs:
                self.distributed_index_bit_swap(pairs)
            self._sync_in()
            local, gz = [], []
            for q, p in pauli.factors:
                bit = self.qubit_map[q]
                if bit < self.local_bits:
                    local.append((bit, p))
                elif p == "Z":
                    gz.append(bit - self.local_bits)
            acc = 0.0 + 0.0j
            for s, st in enumerate(self._devs):
                sign = -1.0 if sum((s >> j) & 1 for j in gz) & 1 else 1.0
                acc += sign * st.expect_pauli(local)
            total += pauli.coefficient * acc
        return total

    # -- verification -------------------------------------------------------------------------
    def to_statevector(self) -> StateVector:
        """Concatenate and undo the qubit map (distsim.py:271-277)."""
        phys = np.concatenate([m.copy() for m in self.segments])
        sv = StateVector.from_amplitudes(phys)
        return StateVector.from_amplitudes(sv.access(self.qubit_map))
