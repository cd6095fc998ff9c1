import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qv, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
n = int(sys.argv[1]); dt = np.complex128 if sys.argv[2] == 'c128' else np.complex64; k = int(sys.argv[3])
ops = fuse_fold(to_gates(gen_qv(n, depth=30, seed=0)), k).ops
sv = StateVector(n, dtype=dt); nat = sv.native
for g in ops[:5]: sv.apply(g)
nat.sync()
nat.prof_enable(True); nat.prof_reset()
t = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
for g in ops: sv.apply(g)
pr.disable()
t_issue = time.perf_counter() - t
nat.sync(); wall = time.perf_counter() - t
prof = nat.prof_read()
kms = sum(v['ms'] for v in prof.values())
print(f"ops {len(ops)} issue {t_issue*1e3:.1f} ms wall {wall*1e3:.1f} ms kernels {kms:.1f} ms", {k2:(v['count'], round(v['ms'],1)) for k2,v in prof.items()})
pstats.Stats(pr).sort_stats('tottime').print_stats(8)
