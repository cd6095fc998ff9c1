import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
n = 30; rng = np.random.default_rng(0)
sv = StateVector(n, dtype=np.complex64)
for q in range(n): sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
m = G.random_unitary(32, rng)
for tg in [(1, 2, 3, 4, 5), (8, 9, 10, 11, 12)]:
    sv.apply(G.DenseGate(m, tg))
sv.native.sync()
