"""BASELINE configs[1]: 30-qubit random circuit of 1- and 2-qubit gates
(complex64), unfused, on one GPU: circuit gates/s and achieved HBM GB/s of
the algorithmic bytes (per-kernel classes from the library's CUDA events)."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import random_gate_sequence
from paper_2308_01999_b200.statevec import StateVector
from tools.sweep import peak

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
gates = random_gate_sequence(n, 200, np.random.default_rng(0), max_arity=2)
sv = StateVector(n, dtype=np.complex64)
nat = sv.native
for g in gates[:10]:
    sv.apply(g)
nat.sync()
nat.prof_reset(); nat.prof_enable(True)
nat.event_record(0)
for g in gates:
    sv.apply(g)
nat.event_record(1)
ms = nat.event_elapsed(0, 1)
prof = nat.prof_read()
alg = sum(v["bytes"] for v in prof.values())
pk = peak()
out = {"config": f"random_gate_sequence({n}, 200, default_rng(0), max_arity=2) complex64, unfused",
       "gates": len(gates), "ms": ms, "gates_per_s": len(gates) / (ms / 1e3),
       "alg_GB": alg / 1e9, "GBps": alg / (ms / 1e3) / 1e9, "frac_of_peak": alg / (ms / 1e3) / 1e9 / pk,
       "kernels": {k: {"count": v["count"], "ms": round(v["ms"], 2),
                       "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] else None}
                   for k, v in prof.items()}}
print(json.dumps(out))
