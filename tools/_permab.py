import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak(); rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
def tm(op, frac, label):
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print(label, f"{ms:.2f} ms alg {frac*16*(1<<n)/ms/1e6/pk:.2f}", flush=True)
tm(G.cx(0, 32), 0.5, "cx c0 t32")
tm(G.cx(0, 5), 0.5, "cx c0 t5")
tm(G.cx(4, 3), 0.5, "cx c4 t3")
tm(G.cx(18, 17), 0.5, "cx c18 t17")
for tg in ((0, 1), (1, 2), (0, 2), (0,), (0, 1, 2), (4, 5, 6), (2, 20)):
    k = len(tg); perm = rng.permutation(1 << k)
    tm(G.PermutationGate(perm, np.ones(1 << k), tg), 1.0, f"perm {tg}")
