"""Device-resident state vector: the drop-in for the reference's
``duetsim.statevec`` (/root/reference/pkg/src/duetsim/statevec.py).

The amplitudes live in B200 HBM inside a libdsv segment; every primitive of
the reference's StateVector (the paper's Table I) runs as a CUDA kernel
through the C ABI.  ``amplitudes`` is a host mirror kept coherent lazily:

* reading it downloads the device state once and hands out the mirror;
* the caller may write into the mirror in place (the reference's tests do
  ``sv.amplitudes[:] = ...``) — the write is noticed (mirror.MirrorArray)
  and the next device operation re-uploads it; plain reads never do;
* any device operation invalidates the mirror.

Logical qubits resolve to physical index bits through ``bit_map``, which
only changes under :meth:`StateVector.swap_index_bits` (statevec.py:311-328).
"""

from __future__ import annotations

import struct
from collections.abc import Sequence
from contextlib import contextmanager

import cmath

import numpy as np

from . import _native as N
from .core import InvalidArgumentError, check_swap_pairs
from .gates import DenseGate, Gate, PauliString, PermutationGate
from .mirror import mirror_of

_DEGENERATE_NORM = 1e-12  # statevec.py:19


def _state_dtype(dtype) -> np.dtype:
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.complex64), np.dtype(np.complex128)):
        raise InvalidArgumentError(f"state dtype must be complex64 or complex128, got {dt}")
    return dt


class StateVector:
    """Length-2^n complex amplitude vector in HBM with a qubit -> index-bit map
    (reference statevec.py:119-351)."""

    def __init__(self, num_qubits: int, dtype=np.complex128, device: int | None = None):
        if num_qubits < 1:
            raise InvalidArgumentError("need at least one qubit")
        self.num_qubits = int(num_qubits)
        self.bit_map = list(range(self.num_qubits))
        self._dev = N.NativeState(self.num_qubits, _state_dtype(dtype), device)  # |0...0>
        self._mirror: np.ndarray | None = None
        self._mirror_valid = False
        self._host_dirty = False

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_amplitudes(cls, amps: np.ndarray, copy: bool = True, device: int | None = None) -> "StateVector":
        """Upload an amplitude array (statevec.py:130-140).  Device memory can
        never alias the caller's array, so ``copy=False`` also copies."""
        amps = np.asarray(amps)
        n = int(amps.size).bit_length() - 1
        if amps.size != 1 << n or n < 1:
            raise InvalidArgumentError("amplitude length must be a power of two")
        dtype = amps.dtype if amps.dtype in (np.complex64, np.complex128) else np.complex128
        sv = cls(n, dtype=dtype, device=device)
        sv._dev.upload(np.ascontiguousarray(amps.reshape(-1), dtype=sv.dtype))
        return sv

    @property
    def dtype(self) -> np.dtype:
        return self._dev.dtype

    @property
    def device(self) -> int:
        return self._dev.device

    @property
    def native(self) -> N.NativeState:
        """The libdsv segment (for benchmarks and the distributed layer)."""
        self._sync_in()
        return self._dev

    # -- host mirror ------------------------------------------------------------
    @property
    def amplitudes(self) -> np.ndarray:
        if not self._mirror_valid:
            if self._mirror is None or self._mirror.dtype != self.dtype:
                self._mirror = np.empty(1 << self.num_qubits, dtype=self.dtype)
            self._dev.download(self._mirror)
            self._mirror_valid = True
        # writes into the handed-out array (in place, through views, np.copyto
        # ...) flag it for upload before the next device operation; reads do not
        return mirror_of(self._mirror, self.mark_host_dirty)

    def mark_host_dirty(self) -> None:
        """The mirror returned by ``amplitudes`` was modified (needed only
        after writes through raw buffers, which MirrorArray cannot see)."""
        if self._mirror is not None and self._mirror_valid:
            self._host_dirty = True

    @amplitudes.setter
    def amplitudes(self, values) -> None:
        values = np.asarray(values)
        if values.size != 1 << self.num_qubits:
            raise InvalidArgumentError("amplitude length does not match the qubit count")
        if values.dtype in (np.complex64, np.complex128) and values.dtype != self.dtype:
            self._dev = N.NativeState(self.num_qubits, values.dtype, self._dev.device)
        self._mirror = np.array(values.reshape(-1), dtype=self.dtype, copy=True)
        self._dev.upload(self._mirror)
        self._mirror_valid = True
        self._host_dirty = False

    def _sync_in(self) -> None:
        if self._host_dirty and self._mirror is not None and self._mirror_valid:
            self._dev.upload(self._mirror)
        self._host_dirty = False

    def _mutated(self) -> None:
        self._mirror_valid = False
        self._host_dirty = False

    # -- helpers ------------------------------------------------------------------
    def _bits(self, qubits: Sequence[int]) -> list[int]:
        for q in qubits:
            if not (0 <= q < self.num_qubits):
                raise InvalidArgumentError(f"qubit {q} out of range")
        return [self.bit_map[q] for q in qubits]

    def _control_bits(self, controls) -> list[tuple[int, int]]:
        self._bits([q for q, _ in controls])
        return [(self.bit_map[q], int(v)) for q, v in controls]

    def norm_squared(self) -> float:
        self._sync_in()
        return self._dev.norm2()

    def copy(self) -> "StateVector":
        self._sync_in()
        sv = StateVector.__new__(StateVector)
        sv.num_qubits = self.num_qubits
        sv.bit_map = list(self.bit_map)
        sv._dev = N.NativeState(self.num_qubits, self.dtype, self._dev.device)
        sv._dev.copy_from(self._dev)
        sv._mirror, sv._mirror_valid, sv._host_dirty = None, False, False
        return sv

    # -- CUDA graphs (extension: the reference has none) -----------------------------
    @contextmanager
    def capture(self):
        """Record the device work of the gates applied inside the block into
        one CUDA graph (include/dsv.h dsv_capture_*).  The gates take effect
        at the end of the block (one graph launch); the yielded Recording
        replays the same sequence later with one launch instead of one host
        call per gate — for small states, where the host's per-gate cost
        (~15 us) exceeds the kernel's.  Reductions, downloads and uploads
        inside the block raise InvalidArgumentError."""
        self._sync_in()
        rec = Recording(self, list(self.bit_map))
        self._dev.capture_begin()
        try:
            yield rec
        except BaseException:
            try:
                self._dev.capture_end().close()
            except Exception:  # pragma: no cover - the original error wins
                pass
            self.bit_map = rec.start_map
            raise
        rec.graph = self._dev.capture_end()
        rec.end_map = list(self.bit_map)
        rec.graph.launch()
        self._mutated()

    def logical_amplitudes(self) -> np.ndarray:
        """Amplitudes with bit q of the index = qubit q (statevec.py:163-167)."""
        if self.bit_map == list(range(self.num_qubits)):
            return self.amplitudes.copy()
        return self.access(self.bit_map)

    # -- Table I primitives -----------------------------------------------------------
    def apply(self, g) -> None:
        if isinstance(g, PermutationGate):
            self.apply_generalized_permutation(g)
        elif isinstance(g, DenseGate):
            self.apply_matrix(g)
        else:
            self._apply_folded(g)

    def _apply_folded(self, op) -> None:
        """Ops of the opt-in fold fuser (fusion_fold.py): phased dense windows
        and SWAP-as-relabel (bit_map only, no data movement)."""
        from .fusion_fold import PhasedDenseGate, QubitSwap

        if isinstance(op, QubitSwap):
            self._bits([op.a, op.b])
            self.bit_map[op.a], self.bit_map[op.b] = self.bit_map[op.b], self.bit_map[op.a]
            return
        if not isinstance(op, PhasedDenseGate):
            raise InvalidArgumentError(f"cannot apply {type(op).__name__}")
        bits = self._bits(op.targets)
        pos = {q: m for m, q in enumerate(op.targets)}
        cross = [(pos[a], self._bits([b])[0], t) for a, b, t in op.cross]
        outside = [(self._bits([b])[0], t) for b, t in op.outside]
        self._sync_in()
        m = np.asarray(op.matrix, dtype=self.dtype)
        try:
            self._dev.apply_matrix_phased(m, bits, cross, outside)
        except RuntimeError as e:
            if "tensor-core path" not in str(e):
                raise
            # 6-qubit window off the tensor path: the phase polynomial as
            # diagonal gates (cross terms on (target, outside) pairs, outside
            # terms on single bits), then the window matrix
            for mpos, b, t in cross:
                self._dev.apply_genperm(np.arange(4), np.array([1, 1, 1, cmath.exp(1j * t)], self.dtype),
                                        [bits[mpos], b])
            for b, t in outside:
                self._dev.apply_genperm(np.arange(2), np.array([1, cmath.exp(1j * t)], self.dtype), [b])
            self._dev.apply_matrix(m, bits)
        self._mutated()

    def apply_matrix(self, g: DenseGate) -> None:
        """Dense gate, matrix cast to the state dtype (statevec.py:177-184)."""
        bits = self._bits(g.targets)
        ctrl = self._control_bits(g.controls)
        self._sync_in()
        self._dev.apply_matrix(np.asarray(g.matrix, dtype=self.dtype), bits, ctrl)
        self._mutated()

    def apply_generalized_permutation(self, g: PermutationGate) -> None:
        """out[perm[j]] = diag[j] * in[j], diag cast to the state dtype
        (statevec.py:186-194); bit-exact with the reference."""
        bits = self._bits(g.targets)
        ctrl = self._control_bits(g.controls)
        self._sync_in()
        self._dev.apply_genperm(g.permutation, np.asarray(g.diagonal, dtype=self.dtype), bits, ctrl)
        self._mutated()

    def apply_pauli_rotation(self, theta: float, pauli: PauliString) -> None:
        """psi <- cos(theta/2) psi - i sin(theta/2) (P psi), in one in-place
        pass (statevec.py:196-207 makes a full copy)."""
        if not pauli.factors:
            raise InvalidArgumentError("empty Pauli string")
        bits = self._bits(pauli.qubits)
        self._sync_in()
        self._dev.pauli_rotation(theta, pauli.coefficient, list(zip(bits, (p for _, p in pauli.factors))))
        self._mutated()

    def probabilities(self, qubits: Sequence[int]) -> np.ndarray:
        """Marginal distribution; entry o has bit j = value of qubits[j]
        (statevec.py:209-213).  float32 for complex64 states, as the reference."""
        if len(set(qubits)) != len(qubits):
            raise InvalidArgumentError("qubits must be distinct")
        bits = self._bits(qubits)
        self._sync_in()
        p = self._dev.marginal(bits)
        return p.astype(np.float32) if self.dtype == np.complex64 else p

    def measure(self, qubits: Sequence[int], random_value: float, collapse: bool = True) -> int:
        """Inverse-CDF measurement with optional collapse (statevec.py:215-238)."""
        if len(set(qubits)) != len(qubits):
            raise InvalidArgumentError("qubits must be distinct")
        bits = self._bits(qubits)
        self._sync_in()
        p64 = self._dev.marginal(bits)
        probs = p64.astype(np.float32) if self.dtype == np.complex64 else p64
        total = probs.sum()
        if total < _DEGENERATE_NORM:
            raise InvalidArgumentError("state norm below 1e-12; cannot measure")
        cdf = np.cumsum(probs / total)
        outcome = min(int(np.searchsorted(cdf, random_value, side="right")), len(probs) - 1)
        if collapse:
            kept = float(p64[outcome])
            if kept <= 0.0:
                raise InvalidArgumentError("measured outcome has zero probability")
            self._dev.collapse(bits, outcome, kept)
            self._mutated()
        return outcome

    def expectation(self, obs: DenseGate | Sequence[PauliString]) -> complex:
        """<psi|O|psi> without modifying the state (statevec.py:240-253)."""
        self._sync_in()
        if isinstance(obs, DenseGate):
            if obs.controls:
                work = self.copy()
                work.apply_matrix(obs)
                return work._dev.inner(self._dev).conjugate()
            return self._dev.expect_matrix(np.asarray(obs.matrix, dtype=self.dtype), self._bits(obs.targets))
        total = 0.0 + 0.0j
        for pauli in obs:
            bits = self._bits(pauli.qubits)
            val = self._dev.expect_pauli(list(zip(bits, (p for _, p in pauli.factors))))
            total += pauli.coefficient * val
        return total

    def sample(self, shots: int, qubit_order: Sequence[int] | None = None, seed: int = 0) -> list[str]:
        """Non-collapsing sampling (statevec.py:255-276).  Variates come from
        the same counter-based Philox stream as the reference; the inverse-CDF
        search runs on the device."""
        if shots < 1:
            raise InvalidArgumentError("shots must be >= 1")
        if qubit_order is None:
            qubit_order = list(range(self.num_qubits - 1, -1, -1))
        bits = self._bits(qubit_order)
        self._sync_in()
        variates = np.random.Generator(np.random.Philox(key=seed)).random(shots)
        outcomes = self._dev.sample(variates).astype(np.int64)
        cols = np.stack([(outcomes >> b) & 1 for b in bits], axis=1) if bits else np.zeros((shots, 0), np.int64)
        chars = np.where(cols == 1, "1", "0")
        return ["".join(row) for row in chars]

    def access(self, bit_ordering: Sequence[int], begin: int = 0, end: int | None = None) -> np.ndarray:
        """Copy out amplitudes re-indexed by ``bit_ordering`` (statevec.py:278-294):
        output index bit b reads current index bit ``bit_ordering[b]``."""
        n = self.num_qubits
        if sorted(bit_ordering) != list(range(n)):
            raise InvalidArgumentError("bit_ordering must be a permutation of all index bits")
        if end is None:
            end = 1 << n
        if not (0 <= begin < end <= 1 << n):
            raise InvalidArgumentError(f"bad range [{begin}, {end})")
        self._sync_in()
        return self._dev.access_get(list(bit_ordering), begin, end)

    def access_set(self, bit_ordering: Sequence[int], begin: int, values: np.ndarray) -> None:
        """Setter counterpart of :meth:`access` (statevec.py:296-309)."""
        n = self.num_qubits
        if sorted(bit_ordering) != list(range(n)):
            raise InvalidArgumentError("bit_ordering must be a permutation of all index bits")
        values = np.asarray(values, dtype=self.dtype).reshape(-1)
        end = begin + values.size
        if not (0 <= begin < end <= 1 << n):
            raise InvalidArgumentError("range exceeds state size")
        self._sync_in()
        self._dev.access_set(list(bit_ordering), begin, values)
        self._mutated()

    def swap_index_bits(self, pairs: Sequence[tuple[int, int]]) -> None:
        """Physically exchange index-bit pairs in place and relabel bit_map so
        the logical state is unchanged (statevec.py:311-328).  Bit-exact."""
        check_swap_pairs(pairs)
        n = self.num_qubits
        for a, b in pairs:
            if a >= n or b >= n:
                raise InvalidArgumentError(f"bit pair ({a}, {b}) exceeds {n} qubits")
        self._sync_in()
        self._dev.swap_bits([(int(a), int(b)) for a, b in pairs])
        self._mutated()
        relabel = {}
        for a, b in pairs:
            relabel[a], relabel[b] = b, a
        self.bit_map = [relabel.get(bit, bit) for bit in self.bit_map]

    # -- serialisation (statevec.py:332-351) --------------------------------------------
    # streamed file I/O: the file is written / read in
    # chunks of DUMP_CHUNK amplitudes gathered on the GPU in logical order, so
    # a 33-qubit state never needs a host copy of the whole vector
    DUMP_CHUNK = 1 << 24

    def logical_chunks(self, chunk: int | None = None):
        """Yield the logical-order amplitudes in consecutive chunks (gathered
        on the GPU), so callers can stream a state larger than host memory."""
        n = self.num_qubits
        chunk = chunk or self.DUMP_CHUNK
        identity = self.bit_map == list(range(n))
        self._sync_in()
        for begin in range(0, 1 << n, chunk):
            end = min(1 << n, begin + chunk)
            if identity:
                yield self._dev.download(begin=begin, count=end - begin)
            else:
                yield self._dev.access_get(list(self.bit_map), begin, end)

    def dump(self, path) -> None:
        """``<Q`` qubit count, then interleaved little-endian float64 (re, im)
        in logical order — always float64, also for complex64 states
        (statevec.py:332-340 format)."""
        with open(path, "wb") as fh:
            fh.write(struct.pack("<Q", self.num_qubits))
            for chunk in self.logical_chunks():
                fh.write(chunk.astype(np.complex128).view("<f8").tobytes())

    @classmethod
    def load(cls, path, device: int | None = None, dtype=np.complex128) -> "StateVector":
        """Inverse of :meth:`dump` (statevec.py:342-351), streamed into HBM;
        ``dtype`` may narrow to complex64 on the device."""
        import os

        with open(path, "rb") as fh:
            (n,) = struct.unpack("<Q", fh.read(8))
            if os.fstat(fh.fileno()).st_size != 8 + (16 << n):
                raise InvalidArgumentError("file length does not match qubit count")
            sv = cls(n, dtype=dtype, device=device)
            for begin in range(0, 1 << n, cls.DUMP_CHUNK):
                count = min(1 << n, begin + cls.DUMP_CHUNK) - begin
                raw = np.frombuffer(fh.read(16 * count), dtype="<f8")
                sv._dev.upload(raw.view(np.complex128).astype(sv.dtype), begin=begin)
        sv._mutated()
        return sv


class Recording:
    """A captured gate sequence of one StateVector (StateVector.capture)."""

    def __init__(self, sv: "StateVector", start_map: list[int]):
        self.sv = sv
        self.start_map = start_map
        self.end_map: list[int] | None = None
        self.graph = None

    def replay(self) -> None:
        """Re-run the recorded device work on the state's current amplitudes.
        The bit_map must be the one the recording started from (the recorded
        kernels address physical bits); afterwards it is the one it ended at."""
        if self.graph is None:
            raise InvalidArgumentError("recording not finished")
        if self.sv.bit_map != self.start_map:
            raise InvalidArgumentError("bit_map differs from the one the recording started with")
        self.sv._sync_in()
        self.graph.launch()
        self.sv.bit_map = list(self.end_map)
        self.sv._mutated()

    def close(self) -> None:
        if self.graph is not None:
            self.graph.close()
            self.graph = None


def run_circuit_sv(gates: Sequence[Gate], num_qubits: int, dtype=np.complex128,
                   device: int | None = None) -> StateVector:
    """Apply a gate list to |0...0> (statevec.py:354-359)."""
    sv = StateVector(num_qubits, dtype=dtype, device=device)
    for g in gates:
        sv.apply(g)
    return sv


# ---------------------------------------------------------------------------
# Module-level "raw kernels" on host arrays (statevec.py:44-113), kept for
# API compatibility: they stage the array through a device segment, run the
# CUDA kernel and copy the result back into the caller's array in place.


def _staged(amps: np.ndarray, n: int) -> N.NativeState:
    if amps.size != 1 << n:
        raise InvalidArgumentError("amplitude array length is not 2^n")
    st = N.NativeState(n, _state_dtype(amps.dtype))
    st.upload(np.ascontiguousarray(amps.reshape(-1)))
    return st


def _write_back(st: N.NativeState, amps: np.ndarray) -> None:
    amps.reshape(-1)[:] = st.download()


def apply_dense_bits(amps: np.ndarray, n: int, matrix: np.ndarray, target_bits: Sequence[int],
                     control_bits: Sequence[tuple[int, int]] = ()) -> None:
    st = _staged(amps, n)
    st.apply_matrix(np.asarray(matrix, dtype=amps.dtype), list(target_bits), list(control_bits))
    _write_back(st, amps)


def apply_permutation_bits(amps: np.ndarray, n: int, permutation: np.ndarray, diagonal: np.ndarray,
                           target_bits: Sequence[int], control_bits: Sequence[tuple[int, int]] = ()) -> None:
    st = _staged(amps, n)
    st.apply_genperm(permutation, np.asarray(diagonal, dtype=amps.dtype), list(target_bits), list(control_bits))
    _write_back(st, amps)


def apply_pauli_product_bits(amps: np.ndarray, n: int, factors: Sequence[tuple[int, str]]) -> None:
    st = _staged(amps, n)
    st.pauli_product([(int(b), p) for b, p in factors])
    _write_back(st, amps)


def marginal_probabilities_bits(amps: np.ndarray, n: int, bits: Sequence[int]) -> np.ndarray:
    st = _staged(amps, n)
    p = st.marginal(list(bits))
    return p.astype(np.float32) if amps.dtype == np.complex64 else p
