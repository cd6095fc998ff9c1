"""Per-op device time of the folded QFT-33 (c64) on one GPU: which window is slow."""
import sys, statistics, json
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from tools.sweep import peak

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dt = np.complex128 if len(sys.argv) > 3 and sys.argv[3] == 'c128' else np.complex64
pk = peak()
ops = fuse_fold(to_gates(gen_qft(n)), k).ops
sv = StateVector(n, dtype=dt)
nat = sv.native
res = {}
for rep in range(3):
    for i, op in enumerate(ops):
        nat.prof_reset(); nat.prof_enable(True)
        nat.event_record(0); sv.apply(op); nat.event_record(1)
        ms = nat.event_elapsed(0, 1)
        pr = nat.prof_read(); nat.prof_enable(False)
        cls = ",".join(sorted(pr)) if pr else "-"
        res.setdefault(i, []).append((ms, cls))
tot = 0.0
for i, op in enumerate(ops):
    ms = statistics.median(m for m, _ in res[i])
    tot += ms
    b = 2 * np.dtype(dt).itemsize * (1 << n)
    tg = getattr(op, 'targets', None) or getattr(op, 'qubits', None)
    print(f"{i:2d} {type(op).__name__:16s} {str(tg):22s} {res[i][0][1]:10s} {ms:8.2f} ms  {b/ms/1e6/pk:5.2f}")
print(f"total {tot:.1f} ms -> {len(to_gates(gen_qft(n)))/tot*1e3:.0f} gates/s")
