"""Complex128 QFT through the fold fuser at k = 4 and k = 5 (per-class kernel ms):

    python tools/qft_c128.py 32
"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for k in (4, 5):
    ops = fuse_fold(to_gates(gen_qft(n)), k).ops
    sv = StateVector(n, dtype=np.complex128)
    nat = sv.native
    for rep in range(2):
        nat.set_basis(0); sv.bit_map = list(range(n)); nat.sync()
        nat.prof_reset(); nat.prof_enable(True)
        nat.event_record(0)
        for o in ops:
            sv.apply(o)
        nat.event_record(1)
        tot = nat.event_elapsed(0, 1)
        prof = nat.prof_read(); nat.prof_enable(False)
    print(f"QFT-{n} c128 fold k={k}: {tot:.0f} ms = {len(to_gates(gen_qft(n)))/(tot/1e3):.0f} gates/s", {c: (v['count'], round(v['ms'], 1)) for c, v in prof.items()}, flush=True)
    del sv, nat
