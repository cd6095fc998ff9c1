#!/usr/bin/env python
"""Where the e2e QFT-33 time goes: fuse / alloc / run / probabilities / free."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector, run_circuit_sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
gates = to_gates(gen_qft(n))
for it in range(3):
    t0 = time.perf_counter(); ops = fuse_fold(gates, 5).ops
    t1 = time.perf_counter(); sv = StateVector(n, dtype=np.complex64); sv.native.sync()
    t2 = time.perf_counter()
    for g in ops: sv.apply(g)
    sv.native.sync()
    t3 = time.perf_counter(); p = sv.probabilities([0, 1, 2, 3])
    t4 = time.perf_counter(); del sv
    t5 = time.perf_counter()
    print(f"fuse {1e3*(t1-t0):.1f} ms  alloc {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f}  probs {1e3*(t4-t3):.1f}  free {1e3*(t5-t4):.1f}  sum {p.sum():.6f}")
