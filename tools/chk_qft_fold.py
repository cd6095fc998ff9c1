import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
for n in (15, 20, 24, 25, 26, 30):
    sv = StateVector(n, dtype=np.complex64)
    ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
    nat = sv.native
    for i, op in enumerate(ops):
        sv.apply(op)
    a = sv.native.download()
    print(n, "norm", float(np.vdot(a, a).real), "maxdev", float(np.abs(np.abs(a) - 2**(-n/2)).max()), [getattr(o,'targets',None) for o in ops if hasattr(o,'targets')][-1])
