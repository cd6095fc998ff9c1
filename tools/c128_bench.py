#!/usr/bin/env python
"""complex128 dense / phased windows (the QV-34 c128 configuration's per-GPU work)."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector
from tools.tc_bench import time_op
from tools.sweep import peak

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
pk = peak()
sv = StateVector(n, dtype=np.complex128)
rng = np.random.default_rng(0)
for k in (1, 2, 3, 4, 5):
    for tg in (list(range(n - k, n)), list(range(10, 10 + k)), list(range(k))):
        g = G.DenseGate(G.random_unitary(1 << k, rng), tuple(tg))
        ms, b = time_op(sv, g)
        print(json.dumps({"k": k, "targets": tg, "GBps": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / pk, 3)}))
