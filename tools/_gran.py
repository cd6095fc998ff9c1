"""n=30 c64: ops whose touched runs are shorter than 128 B (ncu dram bytes vs algorithmic)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
n = 30
sv = StateVector(n, dtype=np.complex64); nat = sv.native
for q in range(n): sv.apply(G.h(q))
nat.sync()
sv.swap_index_bits([(3, 20)])
sv.apply(G.cp(0.3, 4, 3))
sv.apply(G.cp(0.3, 18, 17))
sv.apply(G.cx(0, 29))
sv.apply(G.PermutationGate(np.array([1, 3, 0, 2]), np.ones(4), (0, 1)))
nat.sync()
