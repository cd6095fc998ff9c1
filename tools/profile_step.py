#!/usr/bin/env python
"""One benchmark step (reset + fused QFT-n circuit) with nothing else, for ncu:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py --n 33
    ncu --set full --clock-control none --import-source on -k regex:k_diag -s 10 -c 2 \
        -o gpurun_out/prof_diag python tools/profile_step.py --n 28
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2308_01999_b200.circuits import gen_qft, to_gates  # noqa: E402
from paper_2308_01999_b200.fusion import FusionConfig, fuse  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=33)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--fusion", default="5,6", help="'k,d' reference fuser or 'foldK' fold fuser")
    ap.add_argument("--timed", type=int, default=0, help="extra timed steps (CUDA events)")
    args = ap.parse_args()
    if args.fusion.startswith("fold"):
        from paper_2308_01999_b200.fusion_fold import fuse_fold

        ops = fuse_fold(to_gates(gen_qft(args.n)), int(args.fusion[4:] or 5)).ops
    else:
        k, d = (int(x) for x in args.fusion.split(","))
        ops = fuse(to_gates(gen_qft(args.n)), FusionConfig(k, d)).gates
    sv = StateVector(args.n, dtype=np.complex64 if args.dtype == "c64" else np.complex128)
    nat = sv.native
    for step in range(args.steps + args.timed):
        if step == args.steps:
            nat.event_record(0)
        nat.set_basis(0)
        sv.bit_map = list(range(args.n))
        for g in ops:
            sv.apply(g)
    if args.timed:
        nat.event_record(1)
        ms = nat.event_elapsed(0, 1) / args.timed
        gates = len(gen_qft(args.n))
        print(f"fusion={args.fusion} n={args.n}: {ms:.1f} ms/step, {gates / ms * 1e3:.1f} gates/s, {len(ops)} ops")
    nat.sync()
    print(f"ran {args.steps} step(s) of {len(ops)} fused ops at n={args.n}")


if __name__ == "__main__":
    main()
