#!/usr/bin/env python
"""Benchmark: circuit gates/s and achieved HBM GB/s for the BASELINE workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the config its metric is quoted on):
33-qubit QFT (577 gates) in complex64 (64 GiB state), host gate fusion up to
k = 5 with the phase-folding fuser (fusion_fold.py: 7 dense/phased windows,
SWAPs as relabels; the reference's FusionConfig(5, 6) gives 152 ops and is
timed beside it), run from |0...0> on one B200.  A "step" = reset to |0> +
the whole fused circuit.  At N > 1 the same 33-qubit circuit is sharded over
N GPUs by its top log2 N qubits (strong scaling, as in the paper's
PAPER.md:285-298 table) with batched P2P global<->local exchanges; ONE host
process drives all N GPUs (shard.py, torch-free), so a plain
`python bench.py --gpus N` works (under torchrun rank 0 does it and the other
ranks exit; DSV_BENCH_MULTIPROC=1 selects the one-process-per-GPU layer of
multigpu.py instead).  The N > 1 line also carries BASELINE configs 4 and 5
as `legs`: QV-34 complex128 on 2 / 4 GPUs, random-36 complex64 on 4 / 8 GPUs
with expectation values, and at N = 8 the weak-scaling efficiency
T(random-33, 1 GPU) / T(random-36, 8 GPUs).  On a box with fewer GPUs than N
the segments share the devices ("virtual_devices") and the legs are skipped.

value   = circuit gates (577) / device time per step (CUDA events on the
          state's stream, max over ranks), inputs resident in HBM;
e2e     = the same metric through the public Python API (fuse, streamed into
          run_circuit_sv + StateVector alloc + probabilities read-back),
          host wall clock;
roofline= dominant kernel class: algorithmic bytes / its CUDA-event time vs
          the measured HBM copy peak (MEASURED_PEAKS.json);
cpu_baseline = the CPU oracle port of the reference algorithm on this host.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "gates/sec and achieved HBM GB/s (n=33 c64) at 1/2/4/8 B200 vs CPU ref"
N_QUBITS = 33
FUSION = (5, 6)
# qsim-mgpu on 1x H100, QFT-33 c64 k=5: 577 gates / 1.21 s
PUBLISHED_1GPU_GATES_PER_S = 577 / 1.21
CPU_SAMPLE_QUBITS = 24


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


FOLD_K = 5  # fold fuser window size (<= 5 per the config); k=5 windows run on the tensor cores (tc8.cu)


def fuse_ops(gates, fusion: str):
    """'fold': the engine's phase-folding fuser (fusion_fold.py, windows of
    <= FOLD_K qubits, SWAPs as relabels); 'reference': the reference's own
    FusionConfig(5, 6) windows (fusion.py, 152 ops at n=33)."""
    if fusion == "fold":
        from paper_2308_01999_b200.fusion_fold import fuse_fold

        return fuse_fold(gates, FOLD_K).ops
    from paper_2308_01999_b200.fusion import FusionConfig, fuse

    return fuse(gates, FusionConfig(*FUSION)).gates


def workload(fusion: str = "fold"):
    from paper_2308_01999_b200.circuits import gen_qft, to_gates

    gates = to_gates(gen_qft(N_QUBITS))
    t0 = time.perf_counter()
    ops = fuse_ops(gates, fusion)
    return gates, ops, time.perf_counter() - t0


# ---- clocks sampler ------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu")

    def __init__(self, gpu_index):
        # one index or a list (N > 1: every GPU of the run is sampled)
        self.gpu = ",".join(str(g) for g in sorted(set(gpu_index))) if isinstance(gpu_index, (list, tuple)) else gpu_index
        self.rows: list[list[str]] = []
        self._proc = None
        self._thread = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return self

        def pump():
            for line in self._proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self._thread = threading.Thread(target=pump, daemon=True)
        self._thread.start()
        return self

    def stop(self) -> dict:
        if self._proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self._proc.terminate()
        try:
            self._proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self._proc.kill()
        if self._thread:
            self._thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            if len(r) < 7:
                continue
            try:
                util = float(r[6])
                s = float(r[0])
                m = float(r[1])
            except ValueError:
                continue
            smax.append(m)
            if util >= 50:
                sm.append(s)
            for name, v in zip(names, r[2:6]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows), "samples_under_load": len(sm)}


# ---- CPU baseline: the reference itself (baseline/_ref), else the oracle port ------------------

REF_DIR = ROOT / "baseline" / "_ref"


def _reference_api():
    """The UNMODIFIED reference package installed by tools/install_reference.sh
    into baseline/_ref (git-ignored; it travels to the GPU box with the
    snapshot).  Returns (statevec, fusion, circuits) modules, or None."""
    if not (REF_DIR / "duetsim" / "__init__.py").exists():
        return None
    if "duetsim" in sys.modules and str(REF_DIR) not in str(getattr(sys.modules["duetsim"], "__file__", "")):
        return None  # the repo's drop-in shim is already imported in this process
    sys.path.insert(0, str(REF_DIR))
    import duetsim  # noqa: F401
    from duetsim import circuits, fusion, statevec

    assert str(REF_DIR) in duetsim.__file__, duetsim.__file__
    return statevec, fusion, circuits


def host_info() -> dict:
    info = {"cpu_count": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    try:
        from threadpoolctl import threadpool_info

        info["threadpools"] = [{k: d.get(k) for k in ("internal_api", "num_threads", "version")}
                               for d in threadpool_info()]
    except Exception:  # pragma: no cover - optional
        pass
    return info


def cpu_sample(nq: int, max_ops: int | None = None) -> dict:
    """Time the reference CPU path on QFT-nq fused with FusionConfig(5, 6)
    (complex64) and extrapolate to the 33-qubit workload: per-op time
    x 2^(33-nq) x 152 ops (streaming cost is linear in 2^n beyond the CPU
    caches).  The reference package itself when installed (kind
    "reference"), otherwise the oracle's NumPy restatement ("port")."""
    api = _reference_api()
    if api is not None:
        statevec, fusion, circuits = api
        gates = circuits.to_gates(circuits.gen_qft(nq))
        fc = fusion.fuse(gates, fusion.FusionConfig(*FUSION))
        ops = fc.gates if max_ops is None else fc.gates[:max_ops]
        sv = statevec.StateVector(nq, dtype=np.complex64)
        t0 = time.perf_counter()
        for g in ops:
            sv.apply(g)
        dt = time.perf_counter() - t0
        kind = "reference"
    else:
        from oracle import sv_oracle as O
        from paper_2308_01999_b200.circuits import gen_qft, to_gates
        from paper_2308_01999_b200.fusion import FusionConfig, fuse

        gates = to_gates(gen_qft(nq))
        fc = fuse(gates, FusionConfig(*FUSION))
        ops = fc.gates if max_ops is None else fc.gates[:max_ops]
        amps = np.zeros(1 << nq, dtype=np.complex64)
        amps[0] = 1
        t0 = time.perf_counter()
        for g in ops:
            O.apply_gate(amps, nq, g)
        dt = time.perf_counter() - t0
        kind = "port"
    per_op = dt / len(ops)
    n33_ops = 152  # FusionConfig(5, 6) windows of QFT-33
    t33 = per_op * (1 << (N_QUBITS - nq)) * n33_ops
    return {"value": 577.0 / t33, "unit": "gates/s", "seconds": dt, "ops": len(ops), "per_op_s": per_op,
            "t33_s": t33, "kind": kind, "circuit_gates": len(gates),
            "unextrapolated_gates_per_s": (len(gates) / dt) if max_ops is None else None}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_desc(r: dict, nq: int) -> str:
    who = ("the unmodified reference (baseline/_ref duetsim: fuse + StateVector.apply)" if r["kind"] == "reference"
           else "oracle port (NumPy restatement of statevec.py)")
    return (f"{who} on the full QFT-{nq} fused(5,6) circuit ({r['ops']} ops, {r['seconds']:.1f} s, c64, "
            f"{r['circuit_gates']} circuit gates -> {r['unextrapolated_gates_per_s'] or 0:.1f} gates/s at n={nq}); "
            f"per-op time scaled x2^{N_QUBITS - nq} and x152 ops to QFT-33 (extrapolated: {r['t33_s']:.0f} s "
            f"per circuit)")


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.pop("OPENBLAS_NUM_THREADS", None)  # BLAS on every core, as the reference runs by default
    for _ in range(max(1, min(args.warmup, 1))):
        cpu_sample(CPU_SAMPLE_QUBITS)
    rs = [cpu_sample(CPU_SAMPLE_QUBITS) for _ in range(args.steps)]
    v = statistics.median(r["value"] for r in rs)
    r0 = sorted(rs, key=lambda r: r["value"])[len(rs) // 2]
    line = {
        "metric": METRIC, "value": v, "unit": "gates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(r["seconds"] for r in rs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (QFT circuit from |0>)",
        "config": {"workload": "qft33_c64_fused_k5", "n_qubits": N_QUBITS,
                   "fusion": f"reference FusionConfig{FUSION} (the reference's own fuser)",
                   "sample": f"QFT-{CPU_SAMPLE_QUBITS}, every fused op, per step"},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "gates/s", "cores": cpu_cores(), "kind": r0["kind"],
                         "sample": _cpu_desc(r0, CPU_SAMPLE_QUBITS), "host": host_info()},
        "e2e": {"value": v, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------------------------

def traffic_from_profiles(cls: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(cls)
    except Exception:
        return None


def gate_payload_bytes(gates, itemsize: int) -> int:
    from paper_2308_01999_b200.gates import PermutationGate

    b = 0
    for g in gates:
        if isinstance(g, PermutationGate):
            b += g.diagonal.size * itemsize + g.permutation.size * 8
        elif hasattr(g, "matrix"):
            b += g.matrix.size * itemsize + 16 * (len(getattr(g, "cross", ())) + len(getattr(g, "outside", ())))
    return b


def qft33_check(st, step, ops, samples: int = 1 << 20) -> dict:
    """Correctness of the timed workload at full size (64 GiB, no host copy
    of the state): QFT|0> must be uniform 2^-16.5 and QFT|x> the DFT column
    w^(x y) / sqrt(N), checked on 2^20 amplitudes read back from 16 spread
    chunks (logical indices through the final bit_map), plus the norm and the
    4-qubit marginals.  Bars: north_star max|d| <= 1e-5 absolute; also
    reported relative to the 2^-16.5 amplitude scale."""
    nat = st.native
    n = N_QUBITS
    N = 1 << n
    chunk = samples // 16
    begins = [int(b) for b in np.linspace(0, N - chunk, 16).astype(np.int64)]
    out = {}
    for tag, x in (("qft_zero", 0), ("qft_x", 0x1_2345_6789 % N)):
        nat.set_basis(x)
        st.bit_map = list(range(n))
        for g in ops:
            st.apply(g)
        qubit_of_bit = [0] * n
        for q, b in enumerate(st.bit_map):
            qubit_of_bit[b] = q
        err = 0.0
        for b0 in begins:
            a = nat.download(np.empty(chunk, np.complex64), b0, chunk).astype(np.complex128)
            phys = np.arange(b0, b0 + chunk, dtype=np.uint64)
            logical = np.zeros(chunk, dtype=np.uint64)
            for b in range(n):
                logical |= ((phys >> np.uint64(b)) & np.uint64(1)) << np.uint64(qubit_of_bit[b])
            xy = (logical * np.uint64(x)) & np.uint64(N - 1)  # x*y mod 2^n (uint64 wraps mod 2^64)
            want = np.exp(2j * np.pi * (xy.astype(np.float64) / N)) / np.sqrt(N)
            err = max(err, float(np.abs(a - want).max()))
        p = st.probabilities([0, 1, 2, 3])
        out[tag] = {"x": x, "samples": samples, "max_abs_dev": err, "max_rel_dev": err * np.sqrt(N),
                    "norm_dev": abs(st.norm_squared() - 1.0),
                    "marginal_max_dev": float(np.abs(p - 1 / 16).max())}
    ok = all(v["max_abs_dev"] <= 1e-5 and v["norm_dev"] <= 1e-5 for v in out.values())
    out["pass"] = ok
    if not ok:
        print(json.dumps({"qft33_check": out}), file=sys.stderr, flush=True)
        raise RuntimeError("QFT-33 result check failed")
    return out


def c128_reference_fuser_leg(dev, n: int = 31) -> dict:
    """What a drop-in caller of the reference gets for complex128: quantum
    volume depth 30 through the reference's own fuser (FusionConfig(5, 6),
    mostly 5-qubit windows), on the complex128 tensor-core kernel (tc8d.cu)
    and, for comparison, on the FP64 CUDA cores (dsv_config_set("tc8d", 0))."""
    from paper_2308_01999_b200 import _native as N
    from paper_2308_01999_b200.circuits import gen_qv, to_gates
    from paper_2308_01999_b200.fusion import FusionConfig, fuse
    from paper_2308_01999_b200.statevec import StateVector

    gates = to_gates(gen_qv(n, 30, seed=0))
    ops = fuse(gates, FusionConfig(5, 6)).gates
    sv = StateVector(n, dtype=np.complex128, device=dev)
    nat = sv.native
    out = {"n_qubits": n, "circuit_gates": len(gates), "ops": len(ops),
           "ops_5_qubits": sum(1 for o in ops if len(o.targets) == 5)}
    try:
        for flag, key in ((1, "tensor_cores"), (0, "fp64_cuda_cores")):
            N.config_set("tc8d", flag)
            nat.set_basis(0)
            sv.bit_map = list(range(n))
            sv.apply(ops[0])
            nat.set_basis(0)
            sv.bit_map = list(range(n))
            nat.sync()
            nat.prof_reset()
            nat.prof_enable(True)
            nat.event_record(0)
            for o in ops:
                sv.apply(o)
            nat.event_record(1)
            ms = nat.event_elapsed(0, 1)
            prof = nat.prof_read()
            nat.prof_enable(False)
            out[key] = {"gates_per_s": len(gates) / (ms / 1000.0), "ms_per_circuit": ms,
                        "tensor_windows": prof.get("dense_tc", {}).get("count", 0),
                        "norm_dev": abs(sv.norm_squared() - 1.0)}
    finally:
        N.config_set("tc8d", 1)
        del sv, nat
    out["speedup"] = out["tensor_cores"]["gates_per_s"] / out["fp64_cuda_cores"]["gates_per_s"]
    return out


def run_single(args) -> None:
    from paper_2308_01999_b200 import _native as N
    from paper_2308_01999_b200.statevec import StateVector

    dev = N.default_device()
    gates, ops, fuse_s = workload(args.fusion)
    st = StateVector(N_QUBITS, dtype=np.complex64, device=dev)
    nat = st.native
    ident = list(range(N_QUBITS))

    def step(op_list=ops):
        nat.set_basis(0)
        st.bit_map = list(ident)
        for g in op_list:
            st.apply(g)

    for _ in range(args.warmup):
        step()
    nat.sync()
    nat.prof_reset()
    nat.prof_enable(True)
    clocks = ClockSampler(dev).start()
    time.sleep(0.3)
    launches0 = N.launch_count()
    nat.event_record(0)
    for _ in range(args.steps):
        step()
    nat.event_record(1)
    ms_total = nat.event_elapsed(0, 1)
    launches = N.launch_count() - launches0
    clk = clocks.stop()
    prof = nat.prof_read()
    nat.prof_enable(False)
    nat.prof_reset()
    ms_step = ms_total / args.steps
    value = len(gates) / (ms_step / 1000.0)
    alg_bytes = sum(v["bytes"] for v in prof.values()) / args.steps
    pk = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    dom_name, dom_v = dom
    per_launch_bytes = dom_v["bytes"] / dom_v["count"]
    per_launch_ms = dom_v["ms"] / dom_v["count"]
    achieved = per_launch_bytes / (per_launch_ms / 1000.0) / 1e9
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"],
                "traffic": traffic_from_profiles(dom_name),
                "alg_bytes_per_launch": per_launch_bytes, "launches": dom_v["count"],
                "share_of_step": dom_v["ms"] / ms_total}
    kernels = {k: {"count": v["count"] // args.steps, "ms_per_step": v["ms"] / args.steps,
                   "GB_per_s": (v["bytes"] / (v["ms"] / 1000.0) / 1e9) if v["ms"] else None}
               for k, v in prof.items()}
    # the same state, the reference fuser's 152 windows (drop-in fusion semantics)
    ref_ops = fuse_ops(gates, "reference") if args.fusion == "fold" else ops
    step(ref_ops)
    nat.event_record(2)
    step(ref_ops)
    nat.event_record(3)
    ref_ms = nat.event_elapsed(2, 3)
    # the same circuit with 6-qubit fold windows (one pass fewer; outside the
    # config's k <= 5, reported beside it, not as the value)
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    k6_ops = fuse_fold(gates, 6).ops
    step(k6_ops)
    k6_ms = []
    for _ in range(2):
        nat.event_record(2)
        step(k6_ops)
        nat.event_record(3)
        k6_ms.append(nat.event_elapsed(2, 3))
    k6_ms = min(k6_ms)
    # the same circuit on the fp32-level bf16-limb tensor kernels (tc.cu,
    # DSV_TC8=0): the int8-digit default drops the digit products below 2^16
    N.config_set("tc8", 0)
    step()
    nat.event_record(2)
    step()
    nat.event_record(3)
    tc_ms = nat.event_elapsed(2, 3)
    N.config_set("tc8", 1)
    # generic states (random amplitudes keep the tensor kernels busier and can
    # trip sw_power_cap): quantum volume depth 30 fold-fused at k = 5, and
    # config 5's random 1-/2-qubit generator unfused, both at n = 33 c64
    from paper_2308_01999_b200.circuits import gen_qv, random_gate_sequence, to_gates

    legs = {}
    clocks2 = ClockSampler(dev).start()
    time.sleep(0.2)
    from paper_2308_01999_b200.fusion_cluster import fuse_auto

    qv_gates = to_gates(gen_qv(N_QUBITS, 30, seed=0))
    qv_ops = fuse_auto(qv_gates, FOLD_K).ops  # cluster fuser: 130 windows (fold / reference: 152)
    rnd = random_gate_sequence(N_QUBITS, 200, np.random.default_rng(0), max_arity=2)
    rnd_ops = fuse_auto(rnd, FOLD_K).ops  # the same 200 gates in <= 5-qubit windows
    qv6_ops = fuse_auto(qv_gates, 6).ops  # 6-qubit windows (tc68.cu): 99 windows
    for name, circ, lops in (("qv33_c64_fused5", qv_gates, qv_ops), ("qv33_c64_fused6", qv_gates, qv6_ops),
                             ("random33_c64", rnd, rnd), ("random33_c64_fused5", rnd, rnd_ops)):
        step(lops)
        nat.event_record(2)
        step(lops)
        nat.event_record(3)
        ms = nat.event_elapsed(2, 3)
        legs[name] = {"gates_per_s": len(circ) / (ms / 1000.0), "ms_per_circuit": ms, "circuit_gates": len(circ),
                      "ops": len(lops), "norm_dev": abs(st.norm_squared() - 1.0)}
    legs["clocks"] = clocks2.stop()
    check = qft33_check(st, step, ops)
    del st, nat
    try:
        legs["qv31_c128_reference_fuser"] = c128_reference_fuser_leg(dev)
    except Exception as e:  # a leg must not take the headline down
        legs["qv31_c128_reference_fuser"] = {"error": f"{type(e).__name__}: {e}"[:300]}

    # e2e through the public API: fuse on the host, allocate, run, read back probabilities
    from paper_2308_01999_b200.statevec import run_circuit_sv

    e2e_times = []
    d2h = 0
    for i in range(max(1, min(args.steps, 3)) + 1):
        t0 = time.perf_counter()
        if args.fusion == "fold":
            # windows stream out of the fuser as it closes them: the GPU runs
            # window i while the host fuses window i + 1
            from paper_2308_01999_b200.fusion_fold import fold_ops

            f2 = fold_ops(gates, FOLD_K)
        else:
            f2 = fuse_ops(gates, args.fusion)
        sv = run_circuit_sv(f2, N_QUBITS, dtype=np.complex64, device=dev)
        p = sv.probabilities([0, 1, 2, 3])
        d2h = p.nbytes
        del sv
        dt = time.perf_counter() - t0
        if i > 0:  # first iteration is the e2e warm-up
            e2e_times.append(dt)
    e2e_s = statistics.median(e2e_times)
    h2d = gate_payload_bytes(ops, 8)

    cpu = None
    if not args.skip_cpu:
        os.environ.pop("OPENBLAS_NUM_THREADS", None)
        r = cpu_sample(CPU_SAMPLE_QUBITS)
        cpu = {"value": r["value"], "unit": "gates/s", "cores": cpu_cores(), "kind": r["kind"],
               "sample": _cpu_desc(r, CPU_SAMPLE_QUBITS)}

    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": value / PUBLISHED_1GPU_GATES_PER_S, "dtype": "c64",
        "data": "synthetic (QFT-33 circuit generated on the host, state starts at |0>)",
        "config": {"workload": "qft33_c64_fused_k5", "n_qubits": N_QUBITS, "circuit_gates": len(gates),
                   "fused_ops": len(ops), "fuse_host_s": fuse_s,
                   "fusion": (f"fold: dense windows <= {FOLD_K} qubits with controlled-phase folding, "
                              "SWAP as relabel (fusion_fold.py)") if args.fusion == "fold"
                   else f"reference FusionConfig{FUSION}",
                   "data_passes": sum(1 for o in ops if hasattr(o, "matrix") or hasattr(o, "diagonal")),
                   "reference_fuser_ops": len(ref_ops),
                   "reference_fuser_gates_per_s": len(gates) / (ref_ms / 1000.0),
                   "fold_k6_gates_per_s": len(gates) / (k6_ms / 1000.0),
                   "fp32_level_tc_gates_per_s": len(gates) / (tc_ms / 1000.0),
                   "l2": "state 64 GiB >> 126 MB L2 (no flush needed)", "parallelism": "single segment",
                   "vs_baseline_ref": "qsim-mgpu 1xH100 QFT-33 k=5: 577 gates/1.21 s (PAPER.md:285-288)"},
        "fused_ops_per_s": len(ops) / (ms_step / 1000.0),
        "hbm_gbs_step": alg_bytes / (ms_step / 1000.0) / 1e9,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": len(gates) / e2e_s, "unit": "gates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "seconds_per_step": e2e_s,
                "path": "fuse (streamed: fold_ops feeds run_circuit_sv) + StateVector alloc + run_circuit_sv + probabilities([0..3])"},
        "gpu_launches": launches,
        "clocks": clk,
        "kernels": kernels,
        "check": check,
        "legs": legs,
    }
    print(json.dumps(line), flush=True)


# ---- N > 1: one host process drives N GPUs (shard.py, torch-free) -------------------------------

def _sharded_time(sv, ops, steps: int, warmup: int, reset=True):
    """Device time per step of `ops` on a ShardedStateVector: CUDA events on
    every segment's stream, max over segments (the exchanges join the
    streams, so each span covers the work it waited for)."""
    def step():
        if reset:
            sv.reset()
        sv.run(ops)

    for _ in range(warmup):
        step()
    sv.sync()
    sv.event_record(0)
    for _ in range(steps):
        step()
    sv.event_record(1)
    sv.sync()
    return sv.event_elapsed_max(0, 1) / steps


def _exchange_gbs(profs) -> dict:
    """NVLink-side rate of the masked exchanges: 2 x 16 bytes cross the link
    per exchanged unit (one read + one write of the partner's half)."""
    ms = sum(p.get("exchange", {}).get("ms", 0.0) for p in profs)
    by = sum(p.get("exchange", {}).get("bytes", 0.0) for p in profs)
    if not ms:
        return {"launches": 0}
    return {"launches": int(sum(p.get("exchange", {}).get("count", 0) for p in profs)),
            "ms_sum_over_devices": ms, "hbm_GB_per_s_per_device": by / (ms / 1000.0) / 1e9,
            "link_GB_per_s_per_device_per_direction": by / 4.0 / (ms / 1000.0) / 1e9}


def _run_legs(legs: dict, P: int, devices, shift: int) -> None:
    """BASELINE configs 4 and 5 on the N > 1 run (see run_sharded)."""
    from paper_2308_01999_b200.circuits import gen_qv, random_gate_sequence, to_gates
    from paper_2308_01999_b200.fusion_cluster import fuse_auto
    from paper_2308_01999_b200.gates import PauliString
    from paper_2308_01999_b200.shard import ShardedStateVector

    if P in (2, 4):
        # BASELINE config 4: QV-34 depth 30, complex128 (256 GiB), k = 4 windows
        qv = to_gates(gen_qv(34 - shift, 30, seed=0))
        qv_ops = fuse_auto(qv, 4).ops  # cluster fuser at k = 4: 181 windows (reference: 232)
        s4 = ShardedStateVector(34 - shift, devices, np.complex128)
        s4.prof(True)
        ms = _sharded_time(s4, qv_ops, 1, 1)
        pf = s4.prof_read()
        legs["qv34_c128"] = {"n_qubits": 34 - shift, "gates_per_s": len(qv) / (ms / 1000.0), "ms_per_circuit": ms,
                             "circuit_gates": len(qv), "fused_ops": len(qv_ops),
                             "transfer_stats": s4.stats.as_dict(), "norm": s4.norm_squared(),
                             "exchange": _exchange_gbs(pf)}
        s4.close()
        del s4
    if P in (4, 8):
        # BASELINE config 5: random-36 c64 (512 GiB) + expectation values;
        # weak-scaling efficiency against the same generator at 33 qubits on 1 GPU
        n5 = 36 - shift
        rnd36 = random_gate_sequence(n5, 200, np.random.default_rng(0), max_arity=2)
        s5 = ShardedStateVector(n5, devices, np.complex64)
        s5.prof(True)
        ms36 = _sharded_time(s5, rnd36, 1, 1)
        pf = s5.prof_read()
        t0 = time.perf_counter()
        ev = s5.expectation([PauliString(((0, "Z"), (17, "X"), (n5 - 1, "Y")))])
        zsum = s5.expectation([PauliString(((q, "Z"),)) for q in range(n5)])
        ev_s = time.perf_counter() - t0
        leg = {"n_qubits": n5, "gates_per_s": len(rnd36) / (ms36 / 1000.0), "ms_per_circuit": ms36,
               "circuit_gates": len(rnd36), "transfer_stats": s5.stats.as_dict(),
               "expect_Z0X17Y35": [ev.real, ev.imag], "sum_Zq": zsum.real, "expectation_s": ev_s,
               "norm": s5.norm_squared(), "exchange": _exchange_gbs(pf)}
        s5.close()
        del s5
        # the same 200 gates in <= 5-qubit windows (host fusion is part of the
        # reference pipeline too: its CLI fuses before running)
        rnd36_ops = fuse_auto(rnd36, 5).ops
        s5f = ShardedStateVector(n5, devices, np.complex64)
        ms36f = _sharded_time(s5f, rnd36_ops, 1, 1)
        leg["fused5"] = {"gates_per_s": len(rnd36) / (ms36f / 1000.0), "ms_per_circuit": ms36f,
                         "fused_ops": len(rnd36_ops), "transfer_stats": s5f.stats.as_dict()}
        s5f.close()
        del s5f
        if P == 8:
            rnd33 = random_gate_sequence(n5 - 3, 200, np.random.default_rng(0), max_arity=2)
            s1 = ShardedStateVector(n5 - 3, [devices[0]], np.complex64)
            ms33 = _sharded_time(s1, rnd33, 1, 1)
            s1.close()
            del s1
            leg["weak_scaling"] = {"T33_1gpu_ms": ms33, "T36_8gpu_ms": ms36, "efficiency": ms33 / ms36}
        legs["random36_c64"] = leg


def run_sharded(args) -> None:
    from paper_2308_01999_b200 import _native as N
    from paper_2308_01999_b200.shard import ShardedStateVector

    ndev = N.device_count()
    if ndev < 1:
        raise RuntimeError("bench.py needs a CUDA device")
    P = args.gpus
    virtual = ndev < P
    devices = [d % ndev for d in range(P)]
    gates, ops, fuse_s = workload(args.fusion)
    sv = ShardedStateVector(N_QUBITS, devices, np.complex64)
    clocks = ClockSampler(devices).start()
    time.sleep(0.3)
    sv.prof(True)
    launches0 = N.launch_count()
    ms_step = _sharded_time(sv, ops, args.steps, args.warmup)
    launches = N.launch_count() - launches0
    clk = clocks.stop()
    profs = sv.prof_read()
    sv.prof(False)
    value = len(gates) / (ms_step / 1000.0)
    p = sv.probabilities([0, 1, 2, 3])
    check = {"norm": sv.norm_squared(), "marginal_max_dev_from_1/16": float(np.abs(p - 1 / 16).max())}
    stats = dict(sv.stats.as_dict())
    # dominant gate kernel class summed over devices
    agg: dict[str, dict] = {}
    for pr in profs:
        for k, v in pr.items():
            a = agg.setdefault(k, {"count": 0, "ms": 0.0, "bytes": 0.0})
            for f in a:
                a[f] += v[f]
    pk = peaks()
    dom_name, dom_v = max(((k, v) for k, v in agg.items() if k != "exchange"), key=lambda kv: kv[1]["ms"])
    achieved = (dom_v["bytes"] / dom_v["count"]) / (dom_v["ms"] / dom_v["count"] / 1000.0) / 1e9
    sv.close()
    del sv

    # e2e through the public API: fuse on the host, build, run, read back
    e2e = []
    for i in range(3):
        t0 = time.perf_counter()
        ops2 = fuse_ops(gates, args.fusion)
        sv2 = ShardedStateVector(N_QUBITS, devices, np.complex64)
        sv2.run(ops2)
        pr2 = sv2.probabilities([0, 1, 2, 3])
        sv2.close()
        dt = time.perf_counter() - t0
        if i:
            e2e.append(dt)
    e2e_s = statistics.median(e2e)

    legs = {}
    # DSV_BENCH_LEG_SHIFT=s runs the legs s qubits smaller (functional runs on
    # a 1-GPU box, where the segments share one device)
    shift = int(os.environ.get("DSV_BENCH_LEG_SHIFT", "0"))
    if (not virtual or shift > 0) and not args.skip_legs:
        try:
            _run_legs(legs, P, devices, shift)
        except Exception as e:  # a leg must not cost the main line
            legs["error"] = f"{type(e).__name__}: {e}"[:400]

    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (QFT-33 circuit generated on the host, state starts at |0>)",
        "config": {"workload": "qft33_c64_fused_k5", "n_qubits": N_QUBITS, "circuit_gates": len(gates),
                   "fused_ops": len(ops), "fuse_host_s": fuse_s, "fusion": args.fusion,
                   "global_bits": int(math.log2(P)), "devices": devices, "virtual_devices": virtual,
                   "l2": "segments >= 8 GiB >> 126 MB L2 (no flush needed)",
                   "parallelism": f"sv-shard{P}: one host process drives {P} GPUs (shard.py, torch-free); "
                                  "top log2 P qubits global, batched P2P masked exchanges over NVLink"},
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"],
                     "traffic": traffic_from_profiles(dom_name)},
        "exchange": _exchange_gbs(profs),
        "transfer_stats": stats,
        "check": check,
        "e2e": {"value": len(gates) / e2e_s, "unit": "gates/s", "seconds_per_step": e2e_s,
                "h2d_bytes_per_step": gate_payload_bytes(ops, 8), "d2h_bytes_per_step": int(pr2.nbytes),
                "path": "fuse + ShardedStateVector build + run + probabilities([0..3]), host wall clock"},
        "gpu_launches": launches,
        "clocks": clk,
        "legs": legs,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--fusion", default="fold", choices=["fold", "reference"])
    ap.add_argument("--skip-legs", action="store_true", help="N > 1: skip the config 4 / 5 legs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and os.environ.get("DSV_BENCH_MULTIPROC") == "1":
        # one process per GPU (torch.distributed plumbing, CUDA IPC exchanges)
        from paper_2308_01999_b200 import multigpu

        multigpu.bench_main(args, METRIC, N_QUBITS, FUSION, PUBLISHED_1GPU_GATES_PER_S, workload, ClockSampler,
                            peaks, cpu_cores)
        return
    if world > 1 and int(os.environ.get("RANK", "0")) != 0:
        # launched under torchrun: rank 0 drives every GPU from one host
        # process (shard.py); the other ranks have nothing to do
        return
    if args.gpus > 1:
        run_sharded(args)
        return
    run_single(args)


if __name__ == "__main__":
    main()
