import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak()
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
for pairs in ([(0, 32)], [(0, 1)], [(0, 5)], [(12, 13)]):
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.swap_index_bits(pairs); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print(pairs, f"{ms:.2f} ms alg {8*(1<<n)/ms/1e6/pk:.2f}", flush=True)
