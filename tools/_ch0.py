import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak(); rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
for tg in ((32,), (5,), (3, 9)):
    op = G.DenseGate(G.random_unitary(1 << len(tg), rng), tg, ((0, 1),))
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print("ctl0 dense", tg, f"{ms:.2f} ms alg {8*2*(1<<n)/2/ms/1e6/pk:.2f}", flush=True)
