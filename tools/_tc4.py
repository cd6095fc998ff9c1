import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak(); rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
for tg in ((0, 5, 17, 30), (0, 2, 3, 4), (0, 3, 4, 5), (0, 6, 7, 8), (0, 1, 2, 3), (0, 9, 20, 32)):
    op = G.DenseGate(G.random_unitary(16, rng), tg)
    ts = []
    for _ in range(5):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print("dense4", tg, f"{ms:.2f} ms {16*(1<<n)/ms/1e6/pk:.2f}", flush=True)
