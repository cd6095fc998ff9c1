import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak(); rng = np.random.default_rng(1)
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
for tg, c in (((0, 1), ()), ((1, 2), ()), ((0, 2), ()), ((0, 1, 2), ()), ((1, 2), ((0, 1),)), ((0, 1), ((2, 1),))):
    op = G.DenseGate(G.random_unitary(1 << len(tg), rng), tg, c)
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print("dense", tg, c, f"{ms:.2f} ms full-pass frac {16*(1<<n)/ms/1e6/pk:.2f}", flush=True)
