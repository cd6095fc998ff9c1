import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak()
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
for t, c in ((3, 4), (17, 18), (32, 0), (0, 1), (20, 5)):
    op = G.cp(0.3, c, t)
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print("cp", t, c, f"{ms:.2f} ms {8*2*(1<<n)/4/ms/1e6/pk:.2f}", flush=True)
for t, c in ((32, 0), (5, 0), (17, 0)):
    op = G.cx(c, t)
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print("cx", t, c, f"{ms:.2f} ms alg {8*2*(1<<n)/2/ms/1e6/pk:.2f}", flush=True)
