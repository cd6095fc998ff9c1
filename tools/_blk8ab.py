import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak()
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
def tm(op, label):
    ts = []
    for _ in range(4):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    ms = statistics.median(ts[1:])
    print(label, f"{ms:.2f} ms full-pass frac {16*(1<<n)/ms/1e6/pk:.2f}", flush=True)
tm(G.cx(1, 0), "cx c1 t0")
tm(G.cp(0.3, 1, 0), "cp c1 t0")
tm(G.cp(0.3, 2, 1), "cp c2 t1")
tm(G.cx(0, 2), "cx c0 t2")
tm(G.PermutationGate(np.arange(4), np.exp(1j * np.arange(4)), (0, 1)), "diag (0,1)")
tm(G.PermutationGate(np.arange(2), np.exp(1j * np.arange(2)), (5,)), "diag (5) ref")
tm(G.PermutationGate(np.arange(2), np.exp(1j * np.arange(2)), (2,)), "diag (2) half active")
tm(G.cx(2, 1), "cx c2 t1")
tm(G.PermutationGate(np.array([1, 0]), np.ones(2), (2,)), "x(2)")
