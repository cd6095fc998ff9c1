import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
n=int(sys.argv[1]); bits=[int(x) for x in sys.argv[2].split(',')]
sv=StateVector(n, dtype=np.complex64); sv.apply(G.h(0))
for _ in range(3): sv.probabilities(bits)
