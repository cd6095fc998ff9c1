"""Per-window timing of complex128 k = 5 dense gates at n qubits (default 32)
for several target layouts, with an A/B config switch (default: tc8d on/off):

    python tools/tc8d_probe.py 32 tc8d 1,0
    python tools/tc8d_probe.py 32 tc8d512 1,0
"""
import sys, json
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200 import _native as N
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
key = sys.argv[2] if len(sys.argv) > 2 else 'tc8d'
vals = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [1, 0]
sv = StateVector(n, dtype=np.complex128)
rng = np.random.default_rng(0)
nat = sv.native
for tg in [(0,1,2,3,4),(3,4,5,6,7),(7,8,9,10,11),(20,21,22,23,24),(1,4,9,17,30),(0,5,11,19,28),(2,3,8,15,31)]:
    g = G.DenseGate(G.random_unitary(32, rng), tg)
    for flag in vals:
        N.config_set(key, flag)
        sv.apply(g); nat.sync()
        ts = []
        for _ in range(3):
            nat.event_record(0); sv.apply(g); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
        ms = min(ts)
        print(tg, key, flag, round(ms, 2), 'ms', round(2 * 16 * 2 ** n / (ms / 1e3) / 1e9), 'GB/s', flush=True)
    N.config_set(key, vals[0])
