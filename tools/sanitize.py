"""compute-sanitizer driver for the tensor-core / mbarrier kernels (n = 14).

    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py
    compute-sanitizer --tool memcheck  python tools/sanitize.py

Runs every tcgen05 kernel family once on a small state — tc8 (k = 4/5 int8
digits: pair, row, row2 and contiguous-tile modes, plain and phased), tc68
(k = 6), and with DSV_TC8=0 the bf16-limb tc.cu / tc6.cu — plus the
low-bit, 64-byte-block and exchange kernels, the complex128 tensor-core
kernel (tc8d, 256- and 512-thread layouts), the batched k = 6 / 7 kernel
and a CUDA-graph capture and
replay, and checks each result against the CPU oracle so a silent
corruption under the tool also fails.
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import sv_oracle as O  # noqa: E402
from paper_2308_01999_b200 import gates as G  # noqa: E402
from paper_2308_01999_b200.circuits import gen_qft, to_gates  # noqa: E402
from paper_2308_01999_b200.fusion_fold import fuse_fold  # noqa: E402
from paper_2308_01999_b200.shard import ShardedStateVector  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402


def main():
    n = int(os.environ.get("SAN_N", "14"))
    rng = np.random.default_rng(0)
    st = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    st = (st / np.linalg.norm(st)).astype(np.complex64)
    worst = 0.0
    # dense k = 4..6 at layouts that select each tensor-core copy mode
    for targets in ((2, 3, 4, 5, 6), (0, 1, 2, 3, 4), (0, 3, 5, 8, 11), (1, 4, 6, 9, 12), (3, 4, 5, 6),
                    (0, 2, 5, 7), (2, 4, 6, 8, 10, 12), (0, 1, 2, 3, 4, 5), (0, 3, 6, 9, 11, 13),
                    (1, 3, 5, 8, 10, 12), (0, 1, 4, 7, 9, 12), (0, 1, 6, 9, 12), (1, 2, 4, 6, 8, 10, 13)):
        m = G.random_unitary(1 << len(targets), rng)
        sv = StateVector.from_amplitudes(st)
        sv.apply(G.DenseGate(m, targets))
        want = st.astype(np.complex128)
        O.apply_dense(want, n, m, list(targets))
        worst = max(worst, float(np.abs(sv.amplitudes - want).max()))
    # fold-fused QFT windows (phased, tile-uniform and row-varying), k = 5 and 6
    for k in (5, 6):
        sv = StateVector.from_amplitudes(st)
        for op in fuse_fold(to_gates(gen_qft(n)), k).ops:
            sv.apply(op)
        want = O.run_circuit(to_gates(gen_qft(n)), n, state=st.astype(np.complex128))
        worst = max(worst, float(np.abs(sv.logical_amplitudes() - want).max()))
    # sharded exchange (two segments on one device: both halves, two streams)
    sh = ShardedStateVector(n, [0, 0, 0, 0], np.complex64)
    sh.run(to_gates(gen_qft(n)))
    worst = max(worst, float(np.abs(sh.gather_logical() - O.run_circuit(to_gates(gen_qft(n)), n)).max()))
    sh.close()
    # complex128 k = 5 on the tensor cores (tc8d): both thread layouts, bit 0 free / a target
    from paper_2308_01999_b200 import _native as N

    st2 = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n))
    st2 /= np.linalg.norm(st2)
    worst128 = 0.0
    for t512 in (1, 0):
        N.config_set("tc8d512", t512)
        for targets in ((3, 4, 5, 6, 7), (0, 2, 5, 9, 13), (1, 4, 6, 9, 12), (0, 2, 4, 6, 8, 10)):
            m = G.random_unitary(1 << len(targets), rng)
            sv = StateVector.from_amplitudes(st2)
            sv.apply(G.DenseGate(m, targets))
            want = st2.copy()
            O.apply_dense(want, n, m, list(targets))
            worst128 = max(worst128, float(np.abs(sv.amplitudes - want).max()))
    N.config_set("tc8d512", 1)
    # CUDA-graph capture and replay of a fold-fused QFT (baked per-gate tables)
    sv = StateVector.from_amplitudes(st)
    with sv.capture() as rec:
        for op in fuse_fold(to_gates(gen_qft(n)), 5).ops:
            sv.apply(op)
    sv.amplitudes = st
    sv.bit_map = list(rec.start_map)
    rec.replay()
    want = O.run_circuit(to_gates(gen_qft(n)), n, state=st.astype(np.complex128))
    worst = max(worst, float(np.abs(sv.logical_amplitudes() - want).max()))
    rec.close()
    print(f"sanitize run ok: max|d| {worst:.2e} c64, {worst128:.2e} c128 (DSV_TC8={os.environ.get('DSV_TC8', '1')})")
    assert worst < 1e-5 and worst128 < 1e-12


if __name__ == "__main__":
    main()
