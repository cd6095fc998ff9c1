"""ctypes binding of libdsv.so (the C ABI declared in include/dsv.h).

PyTorch-free.  The library is loaded lazily on first use so that the host-only
modules (gates, fusion, circuits, planning) import on a machine without a
GPU; every state operation then goes through the CUDA library — there is no
CPU fallback, and a missing or unusable library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from functools import lru_cache
from pathlib import Path

import numpy as np

from .core import InvalidArgumentError

_LIB_PATH = Path(__file__).resolve().parent / "libdsv.so"
_lib = None
_lock = threading.Lock()

DSV_OK, DSV_EINVAL, DSV_ECUDA, DSV_ENOMEM, DSV_EUNSUPPORTED = 0, 1, 2, 3, 4
DSV_C64, DSV_C128 = 0, 1
PROF_NCLASS = 24

_vp = C.c_void_p
_i32 = C.c_int32
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64 = C.c_uint64
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_int = C.c_int
_dbl = C.c_double

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "dsv_last_error": [],
    "dsv_version": [],
    "dsv_device_count": [C.POINTER(_int)],
    "dsv_launch_count": [_u64p],
    "dsv_config_set": [C.c_char_p, _int],
    "dsv_state_create": [_int, _int, _int, C.POINTER(_vp)],
    "dsv_pool_release": [_int],
    "dsv_state_destroy": [_vp],
    "dsv_state_info": [_vp, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)],
    "dsv_state_device_ptr": [_vp, C.POINTER(_vp)],
    "dsv_sync": [_vp],
    "dsv_set_basis": [_vp, _u64],
    "dsv_set_zero": [_vp],
    "dsv_upload": [_vp, _u64, _u64, _vp],
    "dsv_download": [_vp, _u64, _u64, _vp],
    "dsv_copy": [_vp, _vp],
    "dsv_apply_matrix": [_vp, _vp, _i32p, _int, _i32p, _i32p, _int],
    "dsv_apply_genperm": [_vp, _i64p, _vp, _i32p, _int, _i32p, _i32p, _int],
    "dsv_apply_matrix_phased": [_vp, _vp, _i32p, _int, _i32p, _i32p, _dp, _int, _i32p, _dp, _int],
    "dsv_apply_pauli_rotation": [_vp, _dbl, _dbl, _dbl, _i32p, C.c_char_p, _int],
    "dsv_apply_pauli_product": [_vp, _i32p, C.c_char_p, _int],
    "dsv_swap_index_bits": [_vp, _i32p, _int],
    "dsv_access_get": [_vp, _i32p, _u64, _u64, _vp],
    "dsv_access_set": [_vp, _i32p, _u64, _u64, _vp],
    "dsv_norm2": [_vp, _dp],
    "dsv_marginal_probs": [_vp, _i32p, _int, _dp],
    "dsv_expect_pauli": [_vp, _i32p, C.c_char_p, _int, _dp],
    "dsv_expect_matrix": [_vp, _vp, _i32p, _int, _dp],
    "dsv_inner": [_vp, _vp, _dp],
    "dsv_collapse": [_vp, _i32p, _int, _u64, _dbl],
    "dsv_scale": [_vp, _dbl],
    "dsv_sample": [_vp, _dp, C.c_int64, _u64p],
    "dsv_exchange_halves": [_vp, _vp, _int, _int, _int],
    "dsv_exchange_all": [_vp, _vp],
    "dsv_exchange_masked": [_vp, _vp, _i32p, _int, _u64, _u64, _int, _int],
    "dsv_exchange_pair": [_vp, _vp, _i32p, _int, _u64, _u64],
    "dsv_stream_join": [_vp, _vp],
    "dsv_group_norm2": [C.POINTER(_vp), _int, _dp],
    "dsv_group_marginal_probs": [C.POINTER(_vp), _int, _i32p, _int, _dp],
    "dsv_group_expect_pauli": [C.POINTER(_vp), _int, _i32p, C.c_char_p, _int, _dp],
    "dsv_ipc_handle": [_vp, _vp],
    "dsv_peer_open": [_int, _int, _int, _vp, C.POINTER(_vp)],
    "dsv_capture_begin": [_vp],
    "dsv_capture_end": [_vp, C.POINTER(_vp)],
    "dsv_graph_launch": [_vp, _vp],
    "dsv_graph_destroy": [_vp],
    "dsv_prof_enable": [_vp, _int],
    "dsv_prof_reset": [_vp],
    "dsv_prof_read": [_vp, _u64p, _dp, _dp],
    "dsv_prof_class_name": [_int],
    "dsv_event_record": [_vp, _int],
    "dsv_event_elapsed": [_vp, _int, _int, C.POINTER(C.c_float)],
}
_RESTYPES = {"dsv_last_error": C.c_char_p, "dsv_prof_class_name": C.c_char_p}


def library_path() -> Path:
    return Path(os.environ.get("DSV_LIBRARY", str(_LIB_PATH)))


def lib():
    """Load libdsv.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        handle = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        ab_build = "DSV_LIBRARY" in os.environ  # an older build for same-box A/B runs may lack newer entries
        for name, argtypes in SIGNATURES.items():
            if ab_build and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = handle
        return _lib


def check(rc: int, what: str = "") -> None:
    if rc == DSV_OK:
        return
    msg = lib().dsv_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == DSV_EINVAL:
        raise InvalidArgumentError(msg)
    if rc == DSV_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libdsv error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


# ---- marshalling helpers -------------------------------------------------------


# Small index lists go straight into ctypes arrays (no NumPy array + ctypes
# cast per argument: ~1 us each, which made the per-gate host cost of small
# states ~15 us of Python against ~6 us in the C library).
def i32(values) -> tuple:
    vals = [int(v) for v in values]
    return vals, ((C.c_int32 * len(vals))(*vals) if vals else None)


@lru_cache(maxsize=512)
def _array_type(ctype, n: int):
    return ctype * n


def i64(values) -> tuple:
    arr = np.ascontiguousarray(values, dtype=np.int64)
    try:
        return arr, _array_type(C.c_int64, arr.size).from_buffer(arr)
    except (TypeError, ValueError, BufferError):  # read-only input: fall back to the address
        return arr, C.cast(C.c_void_p(arr.ctypes.data), _i64p)


def ptr(arr: np.ndarray):
    """Address of a C-contiguous array for a void* parameter (a ctypes view of
    the buffer: no copy, ~0.6 us instead of ~2 us for arr.ctypes.data)."""
    if arr.nbytes == 0:
        return None
    try:
        return _array_type(C.c_char, arr.nbytes).from_buffer(arr)
    except (TypeError, ValueError, BufferError):  # read-only / foreign buffers
        return C.c_void_p(arr.ctypes.data)


def dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.complex64:
        return DSV_C64
    if dt == np.complex128:
        return DSV_C128
    raise InvalidArgumentError(f"unsupported state dtype {dt}; use complex64 or complex128")


def _square(matrix, dtype, k: int) -> np.ndarray:
    """Gate matrix as a contiguous 2^k x 2^k array of the state dtype; the C ABI
    reads exactly 4^k entries, so a wrong shape is rejected here (the
    reference's NumPy matmul raises on it, statevec.py:60)."""
    m = np.ascontiguousarray(matrix, dtype=dtype)
    d = 1 << k
    if m.shape != (d, d):
        raise InvalidArgumentError(f"matrix shape {m.shape} does not match {k} targets (expected ({d}, {d}))")
    return m


def _table(values, dtype, k: int, what: str) -> np.ndarray:
    a = np.ascontiguousarray(values, dtype=dtype).reshape(-1)
    if a.size != 1 << k:
        raise InvalidArgumentError(f"{what} has {a.size} entries; {k} targets need {1 << k}")
    return a


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().dsv_device_count(C.byref(n))
    return n.value if rc == DSV_OK else 0


def pool_release(device: int = -1) -> None:
    """Free the cached state buffers (device < 0: every device)."""
    call("dsv_pool_release", int(device))


def config_set(key: str, value: int) -> None:
    """Kernel-selection switch (include/dsv.h dsv_config_set)."""
    call("dsv_config_set", key.encode(), int(value))


def launch_count() -> int:
    v = C.c_uint64(0)
    lib().dsv_launch_count(C.byref(v))
    return int(v.value)


def default_device() -> int:
    return int(os.environ.get("DUETSIM_DEVICE", "0"))


class NativeState:
    """Owning handle of one device-resident amplitude segment."""

    __slots__ = ("_h", "nbits", "dtype", "device", "__weakref__")

    def __init__(self, nbits: int, dtype, device: int | None = None, _handle=None):
        self.nbits = int(nbits)
        self.dtype = np.dtype(dtype)
        self.device = default_device() if device is None else int(device)
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        check(lib().dsv_state_create(self.device, self.nbits, dtype_code(self.dtype), C.byref(h)),
              "dsv_state_create")
        self._h = h

    @classmethod
    def open_peer(cls, device: int, nbits: int, dtype, handle64: bytes) -> "NativeState":
        buf = C.create_string_buffer(bytes(handle64), 64)
        h = C.c_void_p()
        check(lib().dsv_peer_open(int(device), int(nbits), dtype_code(dtype), buf, C.byref(h)),
              "dsv_peer_open")
        return cls(nbits, dtype, device, _handle=h)

    @property
    def handle(self):
        return self._h

    @property
    def size(self) -> int:
        return 1 << self.nbits

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h is not None and h.value and _lib is not None:
            _lib.dsv_state_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- thin wrappers ------------------------------------------------------------
    def upload(self, arr: np.ndarray, begin: int = 0) -> None:
        arr = np.ascontiguousarray(arr, dtype=self.dtype)
        call("dsv_upload", self._h, begin, arr.size, ptr(arr))

    def download(self, out: np.ndarray | None = None, begin: int = 0, count: int | None = None) -> np.ndarray:
        if count is None:
            count = self.size - begin
        if out is None:
            out = np.empty(count, dtype=self.dtype)
        assert out.flags.c_contiguous and out.dtype == self.dtype and out.size == count
        call("dsv_download", self._h, begin, count, ptr(out))
        return out

    def sync(self) -> None:
        call("dsv_sync", self._h)

    def set_basis(self, index: int = 0) -> None:
        call("dsv_set_basis", self._h, int(index))

    def set_zero(self) -> None:
        call("dsv_set_zero", self._h)

    def copy_from(self, other: "NativeState") -> None:
        call("dsv_copy", self._h, other._h)

    def apply_matrix(self, matrix, targets, controls=()) -> None:
        t, tp = i32(targets)
        m = _square(matrix, self.dtype, len(t))
        cb, cbp = i32([b for b, _ in controls])
        cv, cvp = i32([v for _, v in controls])
        call("dsv_apply_matrix", self._h, ptr(m), tp, len(t), cbp, cvp, len(cb))

    def apply_matrix_phased(self, matrix, targets, cross=(), outside=()) -> None:
        """cross: (target index m, outside bit, theta); outside: (bit, theta)."""
        t, tp = i32(targets)
        m = _square(matrix, self.dtype, len(t))
        ct, ctp = i32([c[0] for c in cross])
        cb, cbp = i32([c[1] for c in cross])
        cth = np.ascontiguousarray([float(c[2]) for c in cross], dtype=np.float64)
        ob, obp = i32([o[0] for o in outside])
        oth = np.ascontiguousarray([float(o[1]) for o in outside], dtype=np.float64)
        call("dsv_apply_matrix_phased", self._h, ptr(m), tp, len(t), ctp, cbp,
             cth.ctypes.data_as(_dp) if cth.size else None, len(ct), obp,
             oth.ctypes.data_as(_dp) if oth.size else None, len(ob))

    def apply_genperm(self, perm, diag, targets, controls=()) -> None:
        t, tp = i32(targets)
        p, pp = i64(_table(perm, np.int64, len(t), "permutation"))
        d = _table(diag, self.dtype, len(t), "diagonal")
        cb, cbp = i32([b for b, _ in controls])
        cv, cvp = i32([v for _, v in controls])
        call("dsv_apply_genperm", self._h, pp, ptr(d), tp, len(t), cbp, cvp, len(cb))

    def pauli_rotation(self, theta: float, coefficient: complex, factors) -> None:
        bits, bp = i32([b for b, _ in factors])
        ps = "".join(p for _, p in factors).encode()
        c = complex(coefficient)
        call("dsv_apply_pauli_rotation", self._h, float(theta), c.real, c.imag, bp, ps, len(bits))

    def pauli_product(self, factors) -> None:
        bits, bp = i32([b for b, _ in factors])
        ps = "".join(p for _, p in factors).encode()
        call("dsv_apply_pauli_product", self._h, bp, ps, len(bits))

    def swap_bits(self, pairs) -> None:
        flat = [x for pr in pairs for x in pr]
        arr, ap = i32(flat)
        call("dsv_swap_index_bits", self._h, ap, len(pairs))

    def norm2(self) -> float:
        out = C.c_double(0.0)
        call("dsv_norm2", self._h, C.byref(out))
        return float(out.value)

    def marginal(self, bits) -> np.ndarray:
        b, bp = i32(bits)
        out = np.zeros(1 << len(b), dtype=np.float64)
        call("dsv_marginal_probs", self._h, bp, len(b), out.ctypes.data_as(_dp))
        return out

    def expect_pauli(self, factors) -> complex:
        bits, bp = i32([b for b, _ in factors])
        ps = "".join(p for _, p in factors).encode()
        out = np.zeros(2, dtype=np.float64)
        call("dsv_expect_pauli", self._h, bp, ps, len(bits), out.ctypes.data_as(_dp))
        return complex(out[0], out[1])

    def expect_matrix(self, matrix, targets) -> complex:
        t, tp = i32(targets)
        m = _square(matrix, self.dtype, len(t))
        out = np.zeros(2, dtype=np.float64)
        call("dsv_expect_matrix", self._h, ptr(m), tp, len(t), out.ctypes.data_as(_dp))
        return complex(out[0], out[1])

    def inner(self, other: "NativeState") -> complex:
        out = np.zeros(2, dtype=np.float64)
        call("dsv_inner", self._h, other._h, out.ctypes.data_as(_dp))
        return complex(out[0], out[1])

    def collapse(self, bits, outcome: int, norm2_kept: float) -> None:
        b, bp = i32(bits)
        call("dsv_collapse", self._h, bp, len(b), int(outcome), float(norm2_kept))

    def scale(self, factor: float) -> None:
        call("dsv_scale", self._h, float(factor))

    def sample(self, variates: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(variates, dtype=np.float64)
        out = np.zeros(v.size, dtype=np.uint64)
        call("dsv_sample", self._h, v.ctypes.data_as(_dp), v.size, out.ctypes.data_as(_u64p))
        return out

    def access_get(self, ordering, begin: int, end: int) -> np.ndarray:
        o, op = i32(ordering)
        out = np.empty(end - begin, dtype=self.dtype)
        call("dsv_access_get", self._h, op, int(begin), int(end), ptr(out))
        return out

    def access_set(self, ordering, begin: int, values: np.ndarray) -> None:
        o, op = i32(ordering)
        v = np.ascontiguousarray(values, dtype=self.dtype)
        call("dsv_access_set", self._h, op, int(begin), v.size, ptr(v))

    def exchange_halves(self, other: "NativeState", local_bit: int, part: int = 0, nparts: int = 1) -> None:
        call("dsv_exchange_halves", self._h, other._h, int(local_bit), int(part), int(nparts))

    def exchange_all(self, other: "NativeState") -> None:
        call("dsv_exchange_all", self._h, other._h)

    def exchange_masked(self, other: "NativeState", lbits, pat_a: int, pat_b: int, part: int = 0,
                        nparts: int = 1) -> None:
        """Slice `part` of the batched exchange self[off|pat_a] <-> other[off|pat_b]."""
        b, bp = i32(lbits)
        call("dsv_exchange_masked", self._h, other._h, bp, len(b), int(pat_a), int(pat_b), int(part), int(nparts))

    def exchange_pair(self, other: "NativeState", lbits, pat_a: int, pat_b: int) -> None:
        """The whole batched exchange, split between both segments' devices."""
        b, bp = i32(lbits)
        call("dsv_exchange_pair", self._h, other._h, bp, len(b), int(pat_a), int(pat_b))

    def join(self, other: "NativeState") -> None:
        """Make this segment's stream wait for the work queued on other's."""
        call("dsv_stream_join", self._h, other._h)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        call("dsv_ipc_handle", self._h, buf)
        return buf.raw

    # -- CUDA graphs ------------------------------------------------------------------
    def capture_begin(self) -> None:
        call("dsv_capture_begin", self._h)

    def capture_end(self) -> "Graph":
        out = _vp()
        call("dsv_capture_end", self._h, C.byref(out))
        return Graph(out.value, self)

    # -- instrumentation ------------------------------------------------------------
    def prof_enable(self, on: bool = True) -> None:
        call("dsv_prof_enable", self._h, 1 if on else 0)

    def prof_reset(self) -> None:
        call("dsv_prof_reset", self._h)

    def prof_read(self) -> dict:
        cnt = np.zeros(PROF_NCLASS, dtype=np.uint64)
        ms = np.zeros(PROF_NCLASS, dtype=np.float64)
        by = np.zeros(PROF_NCLASS, dtype=np.float64)
        call("dsv_prof_read", self._h, cnt.ctypes.data_as(_u64p), ms.ctypes.data_as(_dp),
             by.ctypes.data_as(_dp))
        out = {}
        for c in range(PROF_NCLASS):
            if cnt[c]:
                name = lib().dsv_prof_class_name(c).decode()
                out[name] = {"count": int(cnt[c]), "ms": float(ms[c]), "bytes": float(by[c])}
        return out

    def event_record(self, slot: int) -> None:
        call("dsv_event_record", self._h, int(slot))

    def event_elapsed(self, a: int, b: int) -> float:
        out = C.c_float(0.0)
        call("dsv_event_elapsed", self._h, int(a), int(b), C.byref(out))
        return float(out.value)


# ---- segment groups (one host thread drives every device) ---------------------------


def _handles(states) -> C.Array:
    arr = (_vp * len(states))(*[st._h for st in states])
    return arr


def group_norm2(states) -> np.ndarray:
    """Per-segment |a|^2 sums, all devices reducing at once."""
    out = np.zeros(len(states), dtype=np.float64)
    call("dsv_group_norm2", _handles(states), len(states), out.ctypes.data_as(_dp))
    return out


def group_marginal(states, bits) -> np.ndarray:
    b, bp = i32(bits)
    out = np.zeros((len(states), 1 << len(b)), dtype=np.float64)
    call("dsv_group_marginal_probs", _handles(states), len(states), bp, len(b), out.ctypes.data_as(_dp))
    return out


def group_expect_pauli(states, factors) -> np.ndarray:
    """Per-segment <P> partial sums as complex values."""
    bits, bp = i32([b for b, _ in factors])
    ps = "".join(p for _, p in factors).encode()
    out = np.zeros((len(states), 2), dtype=np.float64)
    call("dsv_group_expect_pauli", _handles(states), len(states), bp, ps, len(bits), out.ctypes.data_as(_dp))
    return out[:, 0] + 1j * out[:, 1]


class Graph:
    """A recorded gate sequence of one NativeState (dsv_capture_* / dsv_graph_*)."""

    def __init__(self, handle, state: NativeState):
        self._h = handle
        self._state = state  # keeps the state (whose pointers the graph holds) alive

    def launch(self) -> None:
        call("dsv_graph_launch", self._h, self._state._h)

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            lib().dsv_graph_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
