import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 31; pk = peak(); rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex128); nat = sv.native
for q in range(n): sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
for tg in [(0, 1, 2, 3), (0, 2, 4, 5), (4, 5, 6, 7), (10, 11, 12, 13)]:
    op = G.DenseGate(G.random_unitary(16, rng), tg)
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print(tg, f"{ms:.2f} ms {32*(1<<n)/ms/1e6/pk:.2f}", flush=True)
