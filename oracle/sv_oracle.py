"""NumPy restatement of the reference state-vector kernels (TEST ORACLE ONLY;
see oracle/__init__.py).  Each function names the reference code it follows.

Layout: a length-2^n vector viewed as an n-dimensional (2,)*n tensor whose
axis a holds index bit n-1-a (little-endian index, reference core.py:3-5).
"""

from __future__ import annotations

import numpy as np


def _axis(n: int, bit: int) -> int:
    return n - 1 - bit


def _subcube(t: np.ndarray, n: int, controls):
    """Fix control axes to their values (statevec.py:26-31)."""
    sel = [slice(None)] * n
    for bit, val in controls:
        sel[_axis(n, bit)] = int(val)
    return t[tuple(sel)]


def _target_axes_after_controls(n: int, targets, controls):
    """Axis of each target once control axes are indexed away (statevec.py:34-41)."""
    gone = sorted(_axis(n, b) for b, _ in controls)
    out = []
    for b in targets:
        a = _axis(n, b)
        out.append(a - sum(1 for c in gone if c < a))
    return out


def _grouped(amps: np.ndarray, n: int, targets, controls):
    """View whose leading axes are the targets, ordered so the flattened
    leading index is the gate index j (bit m of j = targets[m])."""
    t = amps.reshape((2,) * n)
    sub = _subcube(t, n, controls)
    k = len(targets)
    axes = _target_axes_after_controls(n, targets, controls)
    lead = np.moveaxis(sub, axes, list(range(k - 1, -1, -1)))
    return lead, lead.shape[k:]


def apply_dense(amps: np.ndarray, n: int, matrix: np.ndarray, targets, controls=()) -> None:
    """In-place controlled dense gate (statevec.py:44-60)."""
    k = len(targets)
    lead, rest = _grouped(amps, n, targets, controls)
    block = lead.reshape(1 << k, -1)
    lead[...] = (np.asarray(matrix, dtype=amps.dtype) @ block).reshape((2,) * k + rest)


def apply_genperm(amps: np.ndarray, n: int, perm, diag, targets, controls=()) -> None:
    """out[perm[j]] = diag[j] * in[j] per group (statevec.py:63-81)."""
    k = len(targets)
    lead, rest = _grouped(amps, n, targets, controls)
    block = lead.reshape(1 << k, -1)
    res = np.empty_like(block)
    res[np.asarray(perm, dtype=np.int64)] = np.asarray(diag, dtype=amps.dtype)[:, None] * block
    lead[...] = res.reshape((2,) * k + rest)


def apply_pauli_product(amps: np.ndarray, n: int, factors) -> None:
    """Unit-coefficient Pauli product in place (statevec.py:84-104)."""
    t = amps.reshape((2,) * n)
    for bit, p in factors:
        a = _axis(n, bit)
        lo = tuple(0 if i == a else slice(None) for i in range(n))
        hi = tuple(1 if i == a else slice(None) for i in range(n))
        if p == "X":
            t[lo], t[hi] = t[hi].copy(), t[lo].copy()
        elif p == "Y":
            lo_v = t[lo].copy()
            t[lo] = -1j * t[hi]
            t[hi] = 1j * lo_v
        elif p == "Z":
            t[hi] *= -1


def marginal(amps: np.ndarray, n: int, bits) -> np.ndarray:
    """Marginal over `bits`, entry o has bit j = value of bits[j] (statevec.py:107-113)."""
    k = len(bits)
    p = (amps.real * amps.real + amps.imag * amps.imag).reshape((2,) * n)
    lead = np.moveaxis(p, [_axis(n, b) for b in bits], list(range(k - 1, -1, -1)))
    return lead.reshape(1 << k, -1).sum(axis=1)


def pauli_rotation(amps: np.ndarray, n: int, theta: float, factors, coefficient=1.0) -> None:
    """psi <- cos(theta/2) psi - i sin(theta/2) coef (P psi) (statevec.py:196-207)."""
    rot = amps.copy()
    apply_pauli_product(rot, n, factors)
    if coefficient != 1.0:
        rot *= coefficient
    amps *= np.cos(theta / 2)
    amps -= 1j * np.sin(theta / 2) * rot


def expectation_pauli(amps: np.ndarray, n: int, factors, coefficient=1.0) -> complex:
    """coef * <psi|P|psi> (statevec.py:246-253)."""
    rot = amps.copy()
    apply_pauli_product(rot, n, factors)
    return coefficient * complex(np.vdot(amps, rot))


def expectation_dense(amps: np.ndarray, n: int, matrix, targets, controls=()) -> complex:
    """<psi|O|psi> via copy + apply + vdot (statevec.py:241-245)."""
    work = amps.copy()
    apply_dense(work, n, matrix, targets, controls)
    return complex(np.vdot(amps, work))


def swap_index_bits(amps: np.ndarray, n: int, pairs) -> np.ndarray:
    """Physical bit-pair permutation, returns the new array (statevec.py:311-324)."""
    order = list(range(n))
    for a, b in pairs:
        order[a], order[b] = order[b], order[a]
    axes = [_axis(n, order[_axis(n, i)]) for i in range(n)]
    return np.ascontiguousarray(amps.reshape((2,) * n).transpose(axes)).reshape(-1)


def access(amps: np.ndarray, n: int, ordering, begin: int = 0, end: int | None = None) -> np.ndarray:
    """Output index bit b reads current bit ordering[b] (statevec.py:278-294)."""
    if end is None:
        end = 1 << n
    axes = [_axis(n, ordering[_axis(n, a)]) for a in range(n)]
    return amps.reshape((2,) * n).transpose(axes).reshape(-1)[begin:end].copy()


def access_set(amps: np.ndarray, n: int, ordering, begin: int, values) -> None:
    """Setter counterpart (statevec.py:296-309)."""
    values = np.asarray(values, dtype=amps.dtype)
    j = np.arange(begin, begin + values.size, dtype=np.int64)
    src = np.zeros_like(j)
    for b in range(n):
        src |= ((j >> b) & 1) << ordering[b]
    amps[src] = values


def measure(amps: np.ndarray, n: int, bits, random_value: float, collapse: bool = True):
    """Inverse-CDF measurement + collapse (statevec.py:215-238); returns
    (outcome, new_amps)."""
    probs = marginal(amps, n, bits)
    total = probs.sum()
    cdf = np.cumsum(probs / total)
    outcome = min(int(np.searchsorted(cdf, random_value, side="right")), len(probs) - 1)
    if not collapse:
        return outcome, amps
    out = amps.copy()
    idx = np.arange(1 << n)
    keep = np.ones(1 << n, dtype=bool)
    for j, b in enumerate(bits):
        keep &= ((idx >> b) & 1) == ((outcome >> j) & 1)
    out[~keep] = 0
    out /= np.sqrt(np.sum(out.real * out.real + out.imag * out.imag))
    return outcome, out


def sample_indices(amps: np.ndarray, shots: int, seed: int = 0) -> np.ndarray:
    """Physical outcome indices of StateVector.sample (statevec.py:267-272)."""
    probs = amps.real ** 2 + amps.imag ** 2
    cdf = np.cumsum(probs)
    cdf /= cdf[-1]
    v = np.random.Generator(np.random.Philox(key=seed)).random(shots)
    out = np.searchsorted(cdf, v, side="right")
    return np.clip(out, 0, len(probs) - 1)


def apply_gate(amps: np.ndarray, n: int, g, bit_map=None) -> None:
    """Dispatch a gate payload (statevec.py:171-194), qubits -> bits via bit_map."""
    bm = bit_map if bit_map is not None else list(range(n))
    targets = [bm[q] for q in g.targets]
    controls = [(bm[q], v) for q, v in g.controls]
    if hasattr(g, "permutation"):
        apply_genperm(amps, n, g.permutation, g.diagonal, targets, controls)
    else:
        apply_dense(amps, n, g.matrix, targets, controls)


def run_circuit(gates, n: int, dtype=np.complex128, state=None) -> np.ndarray:
    """run_circuit_sv (statevec.py:354-359) on a host array."""
    if state is None:
        amps = np.zeros(1 << n, dtype=dtype)
        amps[0] = 1.0
    else:
        amps = np.array(state, dtype=dtype, copy=True)
    for g in gates:
        apply_gate(amps, n, g)
    return amps


def bit_permute_naive(index: int, pairs) -> int:
    """Per-bit reconstruction of the swapped index (independent of core.py)."""
    where = {}
    for a, b in pairs:
        where[a], where[b] = b, a
    hi = max([index.bit_length()] + [max(p) + 1 for p in pairs])
    return sum(((index >> where.get(b, b)) & 1) << b for b in range(hi))


def full_operator(n: int, matrix: np.ndarray, targets, controls=()) -> np.ndarray:
    """Explicit 2^n x 2^n controlled operator, entry by entry (slow; n <= 8)."""
    dim = 1 << n
    out = np.zeros((dim, dim), dtype=np.complex128)
    for col in range(dim):
        if any(((col >> q) & 1) != v for q, v in controls):
            out[col, col] = 1.0
            continue
        jin = sum(((col >> q) & 1) << m for m, q in enumerate(targets))
        base = col
        for q in targets:
            base &= ~(1 << q)
        for jout in range(1 << len(targets)):
            row = base | sum(((jout >> m) & 1) << q for m, q in enumerate(targets))
            out[row, col] = matrix[jout, jin]
    return out
