import sys, statistics, time
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
nat.sync()
for (t, c) in ((3, 4), (17, 18), (5, 20), (4, 6), (3, 5), (2, 9)):
    op = G.cp(0.3, c, t)
    ts = []
    for _ in range(5):
        nat.sync(); nat.event_record(0); sv.apply(op); nat.event_record(1); nat.sync(); ts.append(nat.event_elapsed(0, 1))
    nat.event_record(0)
    for _ in range(5): sv.apply(op)
    nat.event_record(1); nat.sync()
    b2b = nat.event_elapsed(0, 1) / 5
    t0 = time.perf_counter(); sv.apply(op); th = (time.perf_counter() - t0) * 1e3; nat.sync()
    print(f"cp c{c} t{t}: single {statistics.median(ts):.3f} ms  back-to-back {b2b:.3f} ms  host-call {th:.3f} ms", flush=True)
