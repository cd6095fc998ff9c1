"""BASELINE configs[3] per GPU: quantum-volume circuit (depth 30) in complex128
on one B200 at n = 33 (137 GB; the 34-qubit config shards this per GPU over
2 GPUs), fused with the fold fuser at k = 4 (complex128 k = 5 is FP64-bound on
the CUDA cores): circuit gates/s and achieved HBM GB/s."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qv, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from tools.sweep import peak

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
gates = to_gates(gen_qv(n, depth=30, seed=0))
ops = fuse_fold(gates, k).ops
sv = StateVector(n, dtype=np.complex128)
nat = sv.native
nat.sync()
nat.prof_reset(); nat.prof_enable(True)
nat.event_record(0)
for g in ops:
    sv.apply(g)
nat.event_record(1)
ms = nat.event_elapsed(0, 1)
prof = nat.prof_read()
alg = sum(v["bytes"] for v in prof.values())
pk = peak()
print(json.dumps({"config": f"QV-{n} depth 30 seed 0, complex128, fold fuser k = {k}", "gates": len(gates),
                  "fused_ops": len(ops), "ms": ms, "gates_per_s": len(gates) / (ms / 1e3),
                  "GBps": alg / (ms / 1e3) / 1e9, "frac_of_peak": alg / (ms / 1e3) / 1e9 / pk,
                  "kernels": {k2: {"count": v["count"], "ms": round(v["ms"], 1),
                                   "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] else None}
                              for k2, v in prof.items()}}))
