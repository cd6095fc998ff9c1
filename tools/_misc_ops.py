"""n = 33 complex64 timings of the ops outside the gate sweep (generic state)."""
import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
pk = peak(); n = 33; rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
def t(label, fn, nbytes, reps=4):
    ts = []
    for _ in range(reps):
        nat.event_record(0); fn(); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print(f"{label:42s} {ms:7.2f} ms {nbytes/ms/1e6:6.0f} GB/s {nbytes/ms/1e6/pk:.2f}", flush=True)
N = 1 << n
t("pauli_rotation Z0 X5", lambda: sv.apply_pauli_rotation(0.3, G.PauliString(((0, "Z"), (5, "X")))), 16 * N)
t("pauli_rotation X0", lambda: sv.apply_pauli_rotation(0.3, G.PauliString(((0, "X"),))), 16 * N)
t("pauli_rotation Z3 Z9", lambda: sv.apply_pauli_rotation(0.3, G.PauliString(((3, "Z"), (9, "Z")))), 16 * N)
t("norm_squared", lambda: sv.norm_squared(), 8 * N)
t("sample 1000 shots", lambda: sv.sample(1000, seed=1), 8 * N)
t("expectation dense 2q (3,17)", lambda: sv.expectation(G.DenseGate(G.random_unitary(4, rng), (3, 17), unitary=False)), 8 * N)
t("expectation dense 3q (0,1,2)", lambda: sv.expectation(G.DenseGate(G.random_unitary(8, rng), (0, 1, 2), unitary=False)), 8 * N)
t("expectation dense 4q (5,9,20,30)", lambda: sv.expectation(G.DenseGate(G.random_unitary(16, rng), (5, 9, 20, 30), unitary=False)), 8 * N)
