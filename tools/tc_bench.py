#!/usr/bin/env python
"""Per-op HBM throughput of k = 4/5 complex64 dense and phased windows.

    python tools/tc_bench.py [--n 30]          # tensor-core path (default)
    DSV_TC=0 python tools/tc_bench.py --n 30   # CUDA-core kernels, for A/B

Ops: dense k = 4, 5 on high / mid / low(>=2) targets, k = 2, 3 on the lowest
bits, and every op of the fold-fused QFT-n at k = 3, 4 and 5.  Median of 5
kernel times (the library's per-launch CUDA events on the state's stream)
after 2 warm-ups; GB/s of algorithmic bytes vs MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2308_01999_b200 import gates as G  # noqa: E402
from paper_2308_01999_b200.circuits import gen_qft, to_gates  # noqa: E402
from paper_2308_01999_b200.fusion_fold import fuse_fold  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402
from tools.sweep import entry, peak  # noqa: E402


def time_op(sv, g, reps=5, warm=2):
    """Median kernel time from the library's own per-launch CUDA events (the
    host-side table building of phased ops is excluded), algorithmic bytes."""
    nat = sv.native
    for _ in range(warm):
        sv.apply(g)
    nat.sync()
    ts, byts = [], 0.0
    for _ in range(reps):
        nat.prof_reset()
        nat.prof_enable(True)
        sv.apply(g)
        prof = nat.prof_read()
        nat.prof_enable(False)
        ts.append(sum(v["ms"] for v in prof.values()))
        byts = sum(v["bytes"] for v in prof.values())
    ts.sort()
    return ts[len(ts) // 2], byts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--only", default="", help="substring filter on op labels (profiling)")
    args = ap.parse_args()
    n = args.n
    pk = peak()
    sv = StateVector(n, dtype=np.complex64)
    rng = np.random.default_rng(0)
    out = []
    for k in (4, 5, 6):
        for label, targets in (("high", list(range(n - k, n))), ("mid", list(range(12, 12 + k))),
                               ("low2", list(range(2, 2 + k))), ("spread", [2, 9, 15, 22, 26, n - 1][:k] if k == 6 else [2, 9, 15, 22, n - 1][:k]),
                               ("low0", list(range(k))), ("with0", [0, 7, 13, 20, 25, 28][:k])):
            g = G.DenseGate(G.random_unitary(1 << k, rng), tuple(targets))
            if args.only not in f"dense{k}_{label}":
                continue
            ms, byts = time_op(sv, g)
            out.append(entry(f"dense{k}_{label}", ms, byts, pk, targets=targets))
    for k in (2, 3):
        g = G.DenseGate(G.random_unitary(1 << k, rng), tuple(range(k)))
        if args.only in f"dense{k}_low0":
            ms, byts = time_op(sv, g)
            out.append(entry(f"dense{k}_low0", ms, byts, pk, targets=list(range(k))))
    for k in (3, 4, 5, 6):
        ops = [op for op in fuse_fold(to_gates(gen_qft(n)), k).ops if type(op).__name__ != "QubitSwap"]
        for i, op in enumerate(ops):
            if args.only not in f"qft{n}_fold{k}_op{i}" and not (args.only == "low" and 0 in op.targets):
                continue
            ms, byts = time_op(sv, op)
            out.append(entry(f"qft{n}_fold{k}_op{i}", ms, byts, pk, targets=list(op.targets),
                             kind=type(op).__name__))
    print(json.dumps({"n": n, "dtype": "c64", "DSV_TC": os.environ.get("DSV_TC", "1"), "peak_GBps": pk,
                      "ops": out}, indent=1))


if __name__ == "__main__":
    main()
