"""A/B of cudaLimitMaxL2FetchGranularity on sparse-run ops (diagnostic)."""
import sys, statistics, ctypes
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.statevec import StateVector
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sv = StateVector(n, dtype=np.complex64); nat = sv.native
rt = ctypes.CDLL('libcudart.so.12')
v = ctypes.c_size_t(0)
print("default L2 fetch granularity", rt.cudaDeviceGetLimit(ctypes.byref(v), 5), v.value)
for q in range(n): sv.apply(G.h(q))
qops = fuse_fold(to_gates(gen_qft(n)), 5).ops
ops = [("cp c4 t3", G.cp(0.3, 4, 3)), ("cp c9 t2", G.cp(0.3, 9, 2)), ("cp c1 t0", G.cp(0.3, 1, 0)),
       ("cp c18 t17", G.cp(0.3, 18, 17)), ("cx c1 t0", G.cx(1, 0)), ("dense1 t5", G.h(5)),
       ("dense2 (1,2)", G.DenseGate(np.kron(G.h(0).matrix, G.h(0).matrix), (1, 2))),
       ("qft win0", qops[0]), ("qft win1", qops[1]), ("qft last", qops[-1])]
ops.append(("swap(3,20)", None))
def t(op):
    ts = []
    for _ in range(4):
        nat.event_record(0)
        if op is None: sv.swap_index_bits([(3, 20)])
        else: sv.apply(op)
        nat.event_record(1); ts.append(nat.event_elapsed(0, 1))
    return statistics.median(ts[1:])
for rep in range(2):
    for g in (128, 64, 32, 0):
        r = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(g)); rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        nat.sync()
        print(f"gran set {g} rc {r} -> {v.value}: " + "  ".join(f"{name} {t(op):.3f}" for name, op in ops), flush=True)
