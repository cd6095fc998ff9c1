"""BASELINE.md §4 results table: every BASELINE.json config on this box, GPU
side (engine, CUDA events, algorithmic bytes from the library's per-launch
profile) beside the UNMODIFIED reference (baseline/_ref) on the host cores.

    python tools/configs_table.py > profiles/configs_table_r2.json

GPU rows: config 1 (QFT-20 c128, unfused 220 gates and FusionConfig(5, 6),
each also replayed as one CUDA graph),
config 2 (random-30 c64, 200 gates unfused), config 3 is bench.py's line,
configs 4 / 5 on ONE B200 as their per-GPU share (QV-33 c128 fold k = 4 =
one segment of QV-34 on 2 GPUs; random-33 c64 = one segment of random-36 on
8 GPUs) — the multi-GPU runs themselves are bench.py --gpus N legs.
CPU rows (reference, all host cores for BLAS): config 1 in full; configs 2,
4 and 5 as the first `CPU_GATES` gates of the same generator at a size the
host holds, scaled by 2^(n - n') and the gate count (labelled extrapolated).
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.pop("OPENBLAS_NUM_THREADS", None)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2308_01999_b200.circuits import gen_qft, gen_qv, random_gate_sequence, to_gates  # noqa: E402
from paper_2308_01999_b200.fusion import FusionConfig, fuse  # noqa: E402
from paper_2308_01999_b200.fusion_cluster import fuse_auto  # noqa: E402
from paper_2308_01999_b200.fusion_fold import fuse_fold  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402

PEAK = bench.peaks()["hbm_gbs"]
NOMINAL = 8000.0
CPU_GATES = int(os.environ.get("CPU_GATES", "8"))


def gpu_run(n, ops, dtype, gates_count, reps=2):
    sv = StateVector(n, dtype=dtype)
    nat = sv.native
    for g in ops[: min(len(ops), 8)]:
        sv.apply(g)
    best = None
    for _ in range(reps):
        nat.set_basis(0)
        sv.bit_map = list(range(n))
        nat.sync()
        nat.prof_reset()
        nat.prof_enable(True)
        nat.event_record(0)
        for g in ops:
            sv.apply(g)
        nat.event_record(1)
        ms = nat.event_elapsed(0, 1)
        prof = nat.prof_read()
        nat.prof_enable(False)
        if best is None or ms < best[0]:
            best = (ms, prof)
    ms, prof = best
    alg = sum(v["bytes"] for v in prof.values())
    gbs = alg / (ms / 1e3) / 1e9
    out = {"ms": ms, "gates_per_s": gates_count / (ms / 1e3), "fused_ops_per_s": len(ops) / (ms / 1e3),
           "alg_GB": alg / 1e9, "GBps": gbs, "frac_measured_peak": gbs / PEAK, "frac_nominal_8TBps": gbs / NOMINAL}
    del sv, nat
    return out


def gpu_graph_run(n, ops, dtype, gates_count, reps=20):
    """The same gate sequence recorded once into a CUDA graph
    (StateVector.capture) and replayed: one launch per pass instead of one
    host call per gate — what a small state (config 1) is bound by."""
    sv = StateVector(n, dtype=dtype)
    nat = sv.native
    with sv.capture() as rec:
        for g in ops:
            sv.apply(g)
    times = []
    for _ in range(reps):
        nat.set_basis(0)
        sv.bit_map = list(rec.start_map)
        nat.sync()
        nat.event_record(0)
        rec.replay()
        nat.event_record(1)
        times.append(nat.event_elapsed(0, 1))
    rec.close()
    ms = float(np.median(times))
    return {"ms_median": ms, "ms_min": min(times), "gates_per_s": gates_count / (ms / 1e3),
            "launch": "one CUDA graph per pass (StateVector.capture / Recording.replay)"}


def cpu_ref(n, gates, dtype, full_n=None, full_count=None):
    api = bench._reference_api()
    assert api is not None, "install the reference first: tools/install_reference.sh"
    statevec = api[0]
    sv = statevec.StateVector(n, dtype=dtype)
    t0 = time.perf_counter()
    for g in gates:
        sv.apply(g)
    dt = time.perf_counter() - t0
    out = {"n": n, "gates_timed": len(gates), "seconds": dt, "cores": bench.cpu_cores()}
    if full_n is not None:
        t_full = dt / len(gates) * full_count * 2 ** (full_n - n)
        out.update({"extrapolated_to": {"n": full_n, "gates": full_count}, "seconds_full": t_full,
                    "gates_per_s": full_count / t_full})
    else:
        out["gates_per_s"] = len(gates) / dt
    return out


def to_ref(gates):
    """This package's gate payloads as the reference's own gate objects."""
    import duetsim.gates as RG  # the reference (bench._reference_api() put baseline/_ref first)

    from paper_2308_01999_b200.gates import PermutationGate

    out = []
    for g in gates:
        if isinstance(g, PermutationGate):
            out.append(RG.PermutationGate(g.permutation, g.diagonal, g.targets, g.controls))
        else:
            out.append(RG.DenseGate(g.matrix, g.targets, g.controls))
    return out


def ref_gates(kind, n, **kw):
    """The same circuits built by the REFERENCE's own generators (its gate objects)."""
    statevec, fusion, circuits = bench._reference_api()
    if kind == "qft":
        return circuits.to_gates(circuits.gen_qft(n))
    if kind == "qv":
        return circuits.to_gates(circuits.gen_qv(n, 30, seed=0))
    raise ValueError(kind)


def main():
    rows = {}
    # ---- config 1: QFT-20 complex128
    g1 = to_gates(gen_qft(20))
    f1 = fuse(g1, FusionConfig(5, 6)).gates
    rows["1_qft20_c128"] = {
        "gpu_unfused": gpu_run(20, g1, np.complex128, len(g1), reps=5),
        "gpu_fused_5_6": gpu_run(20, f1, np.complex128, len(g1), reps=5),
        "gpu_unfused_graph": gpu_graph_run(20, g1, np.complex128, len(g1)),
        "gpu_fused_5_6_graph": gpu_graph_run(20, f1, np.complex128, len(g1)),
    }
    if os.environ.get("CONFIGS_ONLY") == "1":
        print(json.dumps(rows, indent=1))
        return
    statevec, fusion, circuits = bench._reference_api()
    rg = ref_gates("qft", 20)
    rows["1_qft20_c128"]["cpu_reference_unfused"] = cpu_ref(20, rg, np.complex128)
    rows["1_qft20_c128"]["cpu_reference_fused_5_6"] = cpu_ref(
        20, fusion.fuse(rg, fusion.FusionConfig(5, 6)).gates, np.complex128)
    # ---- config 2: random-30 complex64, unfused
    g2 = random_gate_sequence(30, 200, np.random.default_rng(0), max_arity=2)
    f2 = fuse_auto(g2, 5)
    rows["2_random30_c64"] = {"gpu": gpu_run(30, g2, np.complex64, len(g2)),
                              "gpu_fused_auto5": gpu_run(30, f2.ops, np.complex64, len(g2)),
                              "fused_windows": f2.data_passes}
    rows["2_random30_c64"]["cpu_reference"] = cpu_ref(26, to_ref(random_gate_sequence(
        26, CPU_GATES, np.random.default_rng(0), max_arity=2)), np.complex64, full_n=30, full_count=200)
    # ---- config 4 per GPU: QV-33 complex128 fold k = 4 (one of the two 2^33 segments of QV-34 on 2 GPUs)
    g4 = to_gates(gen_qv(33, 30, seed=0))
    rows["4_qv33_c128_per_gpu"] = {"gpu_cluster_k4": gpu_run(33, fuse_auto(g4, 4).ops, np.complex128, len(g4), reps=1),
                                   "windows_cluster_k4": fuse_auto(g4, 4).data_passes,
                                   "windows_fold_k4": fuse_fold(g4, 4).data_passes,
                                   # what a drop-in caller gets: the reference fuser's windows (mostly
                                   # 5 qubits, on the complex128 tensor-core kernel tc8d.cu)
                                   "gpu_reference_fuser_5_6": gpu_run(33, fuse(g4, FusionConfig(5, 6)).gates,
                                                                      np.complex128, len(g4), reps=1)}
    rows["4_qv33_c128_per_gpu"]["cpu_reference"] = cpu_ref(
        26, ref_gates("qv", 26)[:CPU_GATES], np.complex128, full_n=34, full_count=510)
    # ---- config 5 per GPU: random-33 complex64 (one of the 8 segments of random-36)
    g5 = random_gate_sequence(33, 200, np.random.default_rng(0), max_arity=2)
    rows["5_random33_c64_per_gpu"] = {"gpu": gpu_run(33, g5, np.complex64, len(g5), reps=1)}
    rows["5_random33_c64_per_gpu"]["cpu_reference"] = cpu_ref(26, to_ref(random_gate_sequence(
        26, CPU_GATES, np.random.default_rng(0), max_arity=2)), np.complex64, full_n=36, full_count=200)
    rows["host"] = bench.host_info()
    rows["peak_GBps_measured"] = PEAK
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
