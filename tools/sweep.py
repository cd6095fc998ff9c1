#!/usr/bin/env python
"""Kernel roofline sweeps on one B200 (SURVEY.md §8d config 2 methodology).

    python tools/sweep.py [--n 30] [--dtype c64] [--what targets,qft,random]

* targets: dense k=1 over every target position t, k=2 pairs (t, t+1),
  k=3 triples, 100 random target sets per k (PAPER.md:209 methodology),
  plus diagonal / permutation / swap kernels — achieved GB/s of algorithmic
  bytes per launch (CUDA events on the state's stream, median of 5 after 2
  warm-ups), vs the measured HBM copy peak.
* qft: every fused op of QFT-n (5,6) timed individually.
Prints one JSON document.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2308_01999_b200 import gates as G  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text())["hbm_gbs"] if p.exists() else 6650.0


def time_op(sv, g, reps=5, warm=2):
    nat = sv.native
    for _ in range(warm):
        sv.apply(g)
    nat.prof_reset()
    nat.prof_enable(True)
    ts = []
    for _ in range(reps):
        nat.event_record(0)
        sv.apply(g)
        nat.event_record(1)
        ts.append(nat.event_elapsed(0, 1))
    prof = nat.prof_read()
    nat.prof_enable(False)
    nat.prof_reset()
    byts = sum(v["bytes"] for v in prof.values()) / reps
    ms = statistics.median(ts)
    return ms, byts


def entry(label, ms, byts, pk, **kw):
    gbs = byts / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    d = {"op": label, "ms": round(ms, 4), "alg_GB": round(byts / 1e9, 3), "GBps": round(gbs, 1),
         "frac": round(gbs / pk, 4)}
    d.update(kw)
    return d


def sweep_targets(n, dtype, pk, rng):
    sv = StateVector(n, dtype=dtype)
    sv.apply(G.h(0))
    out = []
    for k in (1, 2, 3):
        m = G.random_unitary(1 << k, rng)
        for t in range(0, n - k + 1):
            tg = tuple(range(t, t + k))
            ms, b = time_op(sv, G.DenseGate(m, tg))
            out.append(entry(f"dense{k}", ms, b, pk, targets=list(tg)))
        sets = []
        for _ in range(100):
            tg = tuple(int(x) for x in rng.choice(n, size=k, replace=False))
            ms, b = time_op(sv, G.DenseGate(m, tg), reps=3, warm=1)
            sets.append(b / (ms / 1e3) / 1e9)
        out.append({"op": f"dense{k}_random100", "GBps_median": round(statistics.median(sets), 1),
                    "GBps_min": round(min(sets), 1), "GBps_max": round(max(sets), 1),
                    "frac_median": round(statistics.median(sets) / pk, 4)})
    for k in (4, 5):
        m = G.random_unitary(1 << k, rng)
        for tg in (tuple(range(k)), tuple(range(n - k, n)), tuple(range(10, 10 + k))):
            ms, b = time_op(sv, G.DenseGate(m, tg))
            out.append(entry(f"dense{k}", ms, b, pk, targets=list(tg)))
    for k in (1, 2, 6):
        d = np.exp(1j * rng.uniform(0, 6.3, 1 << k))
        for t in (0, 1, 2, 5, 12, n - k):
            tg = tuple(range(t, t + k))
            ms, b = time_op(sv, G.PermutationGate(np.arange(1 << k), d, tg))
            out.append(entry(f"diag{k}", ms, b, pk, targets=list(tg)))
    for t in (0, 3, 17, n - 1):
        c = (t + 1) % n
        ms, b = time_op(sv, G.cp(0.3, c, t))
        out.append(entry("cp", ms, b, pk, targets=[t], control=c))
        ms, b = time_op(sv, G.cx(c, t))
        out.append(entry("cx", ms, b, pk, targets=[t], control=c))
    for k in (2, 3):
        perm = rng.permutation(1 << k)
        d = np.exp(1j * rng.uniform(0, 6.3, 1 << k))
        for t in (0, 4, n - k):
            tg = tuple(range(t, t + k))
            ms, b = time_op(sv, G.PermutationGate(perm, d, tg))
            out.append(entry(f"perm{k}", ms, b, pk, targets=list(tg)))
    nat = sv.native
    for pairs in ([(0, n - 1)], [(3, 20)], [(12, 13)], [(0, 1), (5, n - 2)]):
        ts = []
        nat.prof_reset()
        nat.prof_enable(True)
        for _ in range(4):
            nat.event_record(0)
            sv.swap_index_bits(pairs)
            nat.event_record(1)
            ts.append(nat.event_elapsed(0, 1))
        prof = nat.prof_read()
        nat.prof_enable(False)
        b = sum(v["bytes"] for v in prof.values()) / 4
        out.append(entry("swap_bits", statistics.median(ts[1:]), b, pk, pairs=pairs))
    for bits in ([0], [n - 1], [0, 7, n - 3]):
        ts = []
        for _ in range(4):
            nat.event_record(0)
            sv.probabilities(bits)
            nat.event_record(1)
            ts.append(nat.event_elapsed(0, 1))
        b = sv.dtype.itemsize * (1 << n)
        out.append(entry("probabilities", statistics.median(ts[1:]), b, pk, bits=bits))
    for fac in (((0, "Z"), (5, "X")), ((n - 1, "Y"), (3, "Z"))):
        ts = []
        for _ in range(4):
            nat.event_record(0)
            sv.expectation([G.PauliString(fac)])
            nat.event_record(1)
            ts.append(nat.event_elapsed(0, 1))
        b = sv.dtype.itemsize * (1 << n)
        out.append(entry("expect_pauli", statistics.median(ts[1:]), b, pk, factors=[list(f) for f in fac]))
    return out


def sweep_qft(n, dtype, pk):
    from paper_2308_01999_b200.circuits import gen_qft, to_gates
    from paper_2308_01999_b200.fusion import FusionConfig, fuse

    fc = fuse(to_gates(gen_qft(n)), FusionConfig(5, 6))
    sv = StateVector(n, dtype=dtype)
    out = []
    for g in fc.gates:
        kind = "dense" if isinstance(g, G.DenseGate) else ("diag" if g.is_diagonal else "perm")
        ms, b = time_op(sv, g, reps=3, warm=1)
        out.append(entry(f"{kind}{len(g.targets)}", ms, b, pk, targets=sorted(g.targets),
                         controls=len(g.controls)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--what", default="targets,qft")
    args = ap.parse_args()
    dtype = np.complex64 if args.dtype == "c64" else np.complex128
    pk = peak()
    rng = np.random.default_rng(0)
    doc = {"n": args.n, "dtype": args.dtype, "peak_GBps": pk}
    what = args.what.split(",")
    if "targets" in what:
        doc["targets"] = sweep_targets(args.n, dtype, pk, rng)
    if "qft" in what:
        doc["qft"] = sweep_qft(args.n, dtype, pk)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
