"""Non-gate operations of the path on a generic state:
complex64 n = 33 and complex128 n = 32 (64 GiB each), CUDA-event time of the
public call, algorithmic bytes (reads s*N, read+write 2*s*N), fraction of the
measured copy peak.   python tools/ops_sweep.py > profiles/ops_sweep_r1.json"""
import json, statistics, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak

pk = peak()
out = {"peak_GBps": pk, "rows": []}
for n, dt in ((33, np.complex64), (32, np.complex128)):
    rng = np.random.default_rng(0)
    sv = StateVector(n, dtype=dt); nat = sv.native
    for q in range(n):
        sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
    s = np.dtype(dt).itemsize; N = 1 << n
    def t(label, fn, nbytes, reps=4):
        ts = []
        for _ in range(reps):
            nat.event_record(0); fn(); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
        ms = statistics.median(ts[1:])
        row = {"op": label, "n": n, "dtype": np.dtype(dt).name, "ms": round(ms, 3),
               "alg_GB": round(nbytes / 1e9, 3), "GBps": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / pk, 3)}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    t("norm_squared", lambda: sv.norm_squared(), s * N)
    for bits in ([0], [n - 1], [0, 7, n - 3], [0, 1, 2, 3]):
        t(f"probabilities {bits}", lambda b=bits: sv.probabilities(b), s * N)
    for fac in (((0, "Z"), (5, "X")), ((n - 1, "Y"), (3, "Z")), ((0, "X"),), ((4, "Z"), (9, "Z"))):
        t(f"expectation pauli {fac}", lambda f=fac: sv.expectation([G.PauliString(f)]), s * N)
    t("expectation dense (3, 17)", lambda: sv.expectation(G.DenseGate(G.random_unitary(4, rng), (3, 17), unitary=False)), s * N)
    t("pauli_rotation Z0 X5", lambda: sv.apply_pauli_rotation(0.3, G.PauliString(((0, "Z"), (5, "X")))), 2 * s * N)
    t("pauli_rotation Z3 Z9", lambda: sv.apply_pauli_rotation(0.3, G.PauliString(((3, "Z"), (9, "Z")))), 2 * s * N)
    t("sample 1000 shots", lambda: sv.sample(1000, seed=1), s * N)
    t("swap_index_bits (12, 13)", lambda: sv.swap_index_bits([(12, 13)]), s * N)
    t("access 2^20 amplitudes (bit-reversed order)", lambda: sv.access(list(range(n))[::-1], 0, 1 << 20), s * (1 << 20) * 2)
    del sv, nat
print(json.dumps(out))
