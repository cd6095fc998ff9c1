import sys, os, statistics
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak(); rng = np.random.default_rng(0)
ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
out = []
for i in (0, 1, 5):
    ts = []
    for _ in range(5):
        nat.event_record(0); sv.apply(ops[i]); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    out.append(f"op{i} {16*(1<<n)/statistics.median(ts[1:])/1e6/pk:.2f}")
print(os.environ.get("DSV_LIBRARY", "product"), " ".join(out), flush=True)
