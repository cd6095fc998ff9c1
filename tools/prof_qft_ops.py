"""Run the folded QFT-n (c64, fold k) once per op on a generic state: the
target for `ncu --set full -k regex:k_dense` captures of its window kernels."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(0)
ops = fuse_fold(to_gates(gen_qft(n)), k).ops
sv = StateVector(n, dtype=np.complex64)
for q in range(n):
    sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
for op in ops:
    sv.apply(op)
sv.native.sync()
print("done", len(ops))
