import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n=33; pk=peak()
ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
sv = StateVector(n, dtype=np.complex64); nat=sv.native
def t(op, label):
    ts=[]
    for _ in range(3):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0,1))
    print(label, [f"{16*(1<<n)/m/1e6/pk:.2f}" for m in ts])
t(ops[0], "op0 on |0> (then evolving)")
t(ops[5], "op5 ")
t(ops[6], "op6 ")
for q in range(n): sv.apply(G.h(q))
rng=np.random.default_rng(0)
for q in range(0,n,5): sv.apply(G.DenseGate(G.random_unitary(2, rng) if hasattr(G,'random_unitary') else np.eye(2), (q,)))
t(ops[0], "op0 generic")
t(ops[1], "op1 generic")
t(ops[5], "op5 generic")
t(ops[6], "op6 generic")
