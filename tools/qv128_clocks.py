"""QV-33 complex128 (cluster k = 4 and the reference fuser) with SM clocks sampled during the run:

    python tools/qv128_clocks.py
"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2308_01999_b200.circuits import gen_qv, to_gates
from paper_2308_01999_b200.fusion import FusionConfig, fuse
from paper_2308_01999_b200.fusion_cluster import fuse_auto
from paper_2308_01999_b200.statevec import StateVector
n = 33
g = to_gates(gen_qv(n, 30, seed=0))
sv = StateVector(n, dtype=np.complex128)
nat = sv.native
for name, ops in (("cluster k4", fuse_auto(g, 4).ops), ("reference fuser (5,6)", fuse(g, FusionConfig(5, 6)).gates)):
    nat.set_basis(0); sv.bit_map = list(range(n)); nat.sync()
    cs = bench.ClockSampler(0).start()
    time.sleep(0.2)
    nat.event_record(0)
    for o in ops:
        sv.apply(o)
    nat.event_record(1)
    ms = nat.event_elapsed(0, 1)
    clk = cs.stop()
    print(name, len(ops), 'ops', round(ms), 'ms', round(len(g) / (ms / 1e3), 1), 'gates/s', clk, flush=True)
