"""One complex128 k = 5 window at n qubits on a random state (ncu target):

    ncu -k regex:k_dense_tc8d -c 1 python tools/tc8d_one.py 28 3,4,5,6,7
"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector
n = int(sys.argv[1]); tg = tuple(int(x) for x in sys.argv[2].split(','))
sv = StateVector(n, dtype=np.complex128)
rng = np.random.default_rng(0)
sv.amplitudes = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / 2 ** (n / 2 + 0.5)
g = G.DenseGate(G.random_unitary(32, rng), tg)
for _ in range(2):
    sv.apply(g)
sv.native.sync()
