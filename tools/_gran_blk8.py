"""n=28 c64: one 64-byte-block permutation and one 64-byte-block dense gate (ncu --set full target)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
n = 28
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
sv.apply(G.PermutationGate(np.array([1, 3, 0, 2]), np.exp(1j * np.arange(4)), (0, 1)))
sv.apply(G.DenseGate(G.random_unitary(4, np.random.default_rng(0)), (1, 2)))
nat.sync()
