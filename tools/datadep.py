"""Does gate throughput depend on the amplitudes?  Same ops on a uniform
state (H on every qubit: all amplitudes equal) and on a generic one (random
1-qubit unitaries on every qubit), with nvidia-smi clocks / power sampled."""
import sys, statistics
sys.path.insert(0, '.')
import numpy as np
from bench import ClockSampler
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from tools.sweep import peak
n = 33; pk = peak()
rng = np.random.default_rng(0)
ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
u1 = G.DenseGate(G.random_unitary(2, rng), (12,))
u1l = G.DenseGate(G.random_unitary(2, rng), (0,))
sv = StateVector(n, dtype=np.complex64); nat = sv.native
def t(op, label, reps=6):
    ts = []
    cs = ClockSampler(0).start()
    for _ in range(reps):
        nat.event_record(0); sv.apply(op); nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    c = cs.stop()
    print(f"{label:28s}", " ".join(f"{16*(1<<n)/m/1e6/pk:.2f}" for m in ts), c, flush=True)
for q in range(n): sv.apply(G.h(q))
t(u1, "uniform 1q t12"); t(u1, "after (still structured)")
for q in range(n): sv.apply(G.h(q))
t(u1l, "uniform 1q t0")
t(ops[1], "uniform op1 tc phased")
for q in range(n): sv.apply(G.DenseGate(G.random_unitary(2, rng), (q,)))
t(u1, "generic 1q t12"); t(u1l, "generic 1q t0")
t(ops[0], "generic op0 tc plain"); t(ops[1], "generic op1 tc phased"); t(ops[5], "generic op5"); t(ops[6], "generic op6 low")
