"""Command-line harness for the B200 engine: ``simulate`` on the state-vector
engines, mirroring the reference's ``duetsim simulate``
(cli.py:124-244) — same flags, same JSON report schema (schema_version,
command, engine, params, counters, digest, verification, timings; timing
fields isolated under "timings" so reports compare equal modulo timings) and
exit codes (0 ok, 2 verification failure or invalid argument, with
``{"error": "invalid-argument", "detail": ...}`` on stderr as in the
reference's cli.py:601-610; ``--workers`` defaults to $DUETSIM_WORKERS,
cli.py:53-54) — extended with what the GPU engine adds: ``--dtype``,
``--fusion fold:K`` (the phase-folding fuser), ``--device``, ``--gpus N``
(the state sharded over N GPUs by one host process, shard.py) and, in the
report, per-kernel-class device times, algorithmic HBM bytes and achieved
GB/s.

``--verify`` follows the reference (cli.py:120-122, :187-210): the result is
compared with the UNFUSED circuit run by the state-vector engine in
complex128 — here that run takes the 1-/2-qubit CUDA-core kernels while the
fused / folded / sharded run under test takes the window and tensor-core
kernels and the exchanges.

    python -m paper_2308_01999_b200.cli simulate --circuit qft --n 30 --dtype c64 --fusion fold:5

The tensor-network, MPS and path-finding commands of the reference are out of
scope for this engine; asking for them is an error.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

from .circuits import Circuit, gen_qaoa_maxcut, gen_qft, gen_qv, to_gates
from .core import InvalidArgumentError
from .distsim import SegmentedStateVector
from .fusion import FusionConfig, fuse
from .statevec import StateVector

REPORT_SCHEMA_VERSION = 1
EXIT_OK = 0
EXIT_VERIFY = 2
DTYPES = {"c64": np.complex64, "c128": np.complex128}
STREAM_QUBITS = 26  # above this the report's digest and norm are streamed chunk by chunk
VERIFY_MAX_QUBITS = 20  # the reference stops at 14 (cli.py:188); the GPU engine verifies up to 20


def default_workers() -> int:
    """Worker count default, as the reference's cli.py:53-54."""
    return int(os.environ.get("DUETSIM_WORKERS", "1"))


def digest_array(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def make_report(command: str, **fields) -> dict:
    report = {"schema_version": REPORT_SCHEMA_VERSION, "command": command}
    report.update(fields)
    report.setdefault("timings", {})
    return report


def emit(report: dict, path: str | None) -> None:
    text = json.dumps(report, indent=2, sort_keys=True)
    if path:
        with open(path, "w") as fh:
            fh.write(text + "\n")
    print(text)


def load_circuit(args) -> Circuit:
    if args.circuit_file:
        return Circuit.load(args.circuit_file)
    if args.circuit == "qft":
        return gen_qft(args.n)
    if args.circuit == "qv":
        return gen_qv(args.n, depth=args.depth, seed=args.seed)
    if args.circuit == "qaoa":
        return gen_qaoa_maxcut([(q, (q + 1) % args.n) for q in range(args.n)], p=args.p, seed=args.seed)
    raise InvalidArgumentError(f"unknown circuit {args.circuit!r}")


def fused_ops(args, gates, counters: dict, timings: dict):
    """Reference FusionConfig windows (--max-fused-*), or the fold fuser (--fusion fold:K)."""
    t0 = time.perf_counter()
    if args.fusion:
        kind, _, k = args.fusion.partition(":")
        if kind not in ("fold", "cluster", "auto"):
            raise InvalidArgumentError(f"unknown fusion {args.fusion!r} (use fold:K, cluster:K or auto:K)")
        from .fusion_cluster import fuse_auto, fuse_cluster
        from .fusion_fold import fuse_fold

        fc = {"fold": fuse_fold, "cluster": fuse_cluster, "auto": fuse_auto}[kind](gates, int(k or 5))
        ops = fc.ops
        counters["data_passes"] = fc.data_passes
    elif args.max_fused_gate_size or args.max_fused_diagonal_gate_size:
        fc = fuse(gates, FusionConfig(max_fused_gate_size=args.max_fused_gate_size or 4,
                                      max_fused_diagonal_gate_size=args.max_fused_diagonal_gate_size or 6))
        ops = fc.gates
    else:
        return gates
    timings["fusion_s"] = time.perf_counter() - t0
    counters["fused_gates"] = len(ops)
    return ops


def _kernel_report(profs: list[dict], seconds: float) -> dict:
    agg: dict = {}
    for prof in profs:
        for name, v in prof.items():
            a = agg.setdefault(name, {"launches": 0, "ms": 0.0, "alg_bytes": 0.0})
            a["launches"] += v["count"]
            a["ms"] += v["ms"]
            a["alg_bytes"] += v["bytes"]
    for a in agg.values():
        a["GB_per_s"] = a["alg_bytes"] / (a["ms"] / 1e3) / 1e9 if a["ms"] > 0 else None
    total_bytes = sum(a["alg_bytes"] for a in agg.values())
    return {"kernels": agg, "alg_bytes": total_bytes,
            "hbm_GB_per_s": total_bytes / seconds / 1e9 if seconds > 0 else None}


def cmd_simulate(args) -> int:
    t_start = time.perf_counter()
    if args.engine not in ("sv", "sv-dist"):
        raise InvalidArgumentError(f"engine {args.engine!r} is not part of the B200 state-vector engine")
    circuit = load_circuit(args)
    n = circuit.num_qubits
    dtype = DTYPES[args.dtype]
    counters: dict = {"gates": len(circuit)}
    timings: dict = {}
    params = {"circuit": args.circuit or args.circuit_file, "n": n, "seed": args.seed, "dtype": args.dtype,
              "global_bits": args.global_bits if args.engine == "sv-dist" else None,
              "workers": args.workers if args.engine == "sv-dist" else None, "fusion": args.fusion}
    if args.dry_run:
        report = make_report("simulate", engine=args.engine, params=params, counters=counters, digest=None)
        report["timings"]["wall_s"] = time.perf_counter() - t_start
        emit(report, args.out)
        return EXIT_OK

    if args.verify and n > VERIFY_MAX_QUBITS:
        raise InvalidArgumentError(f"--verify limited to n <= {VERIFY_MAX_QUBITS}")
    if args.gpus < 1:
        raise InvalidArgumentError("--gpus must be >= 1")
    ops = fused_ops(args, to_gates(circuit), counters, timings)
    if args.engine == "sv" and args.gpus > 1:
        from . import _native as N
        from .shard import ShardedStateVector

        ndev = max(1, N.device_count())
        devices = [d % ndev for d in range(args.gpus)]
        t0 = time.perf_counter()
        sh = ShardedStateVector(n, devices, dtype)
        timings["alloc_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        sh.prof(True)
        sh.run(ops)
        sh.sync()
        timings["apply_s"] = time.perf_counter() - t0
        counters.update(_kernel_report(sh.prof_read(), timings["apply_s"]))
        counters["transfer_stats"] = sh.stats.as_dict()
        params["gpus"] = args.gpus
        amps = sh.gather_logical()
        sh.close()
    elif args.engine == "sv":
        t0 = time.perf_counter()
        sv = StateVector(n, dtype=dtype, device=args.device)
        sv.native.sync()
        timings["alloc_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        nat = sv.native
        nat.prof_enable(True)
        for g in ops:
            sv.apply(g)
        nat.sync()
        timings["apply_s"] = time.perf_counter() - t0
        counters.update(_kernel_report([nat.prof_read()], timings["apply_s"]))
        nat.prof_enable(False)
        if n > STREAM_QUBITS:
            # stream the digest and norm: no host copy of the whole state
            h = hashlib.sha256()
            norm = 0.0
            for chunk in sv.logical_chunks():
                c64 = chunk.astype(np.complex128)
                norm += float(np.vdot(c64, c64).real)
                h.update(np.ascontiguousarray(np.round(c64, 12)).tobytes())
            counters["norm"] = norm
            report = make_report("simulate", engine=args.engine, params=params, counters=counters,
                                 digest=h.hexdigest(), verification=None)
            timings["kernels"] = counters.pop("kernels")
            timings["hbm_GB_per_s"] = counters.pop("hbm_GB_per_s")
            report["timings"] = timings
            report["timings"]["wall_s"] = time.perf_counter() - t_start
            emit(report, args.out)
            return EXIT_OK
        amps = sv.logical_amplitudes()
    else:
        t0 = time.perf_counter()
        devices = None
        if args.gpus > 1:
            from . import _native as N

            devices = [d % max(1, N.device_count()) for d in range(args.gpus)]
            params["gpus"] = args.gpus
        with SegmentedStateVector(n, args.global_bits, args.workers, dtype=dtype, devices=devices) as ssv:
            segs = ssv.native_segments
            for s in segs:
                s.prof_enable(True)
            ssv.run(ops)
            for s in segs:
                s.sync()
            timings["apply_s"] = time.perf_counter() - t0
            counters.update(_kernel_report([s.prof_read() for s in segs], timings["apply_s"]))
            counters["transfer_stats"] = ssv.transfer_stats().as_dict()
            amps = ssv.to_statevector().amplitudes
    a64 = amps.astype(np.complex128)  # float64 sum: a float32 vdot stalls near 2^-24 relative at n >= 28
    counters["norm"] = float(np.vdot(a64, a64).real)
    digest = digest_array(np.round(a64, 12))

    verification = None
    if args.verify:
        # the unfused circuit in complex128 on the same engine (the reference
        # verifies against its own run_circuit_sv the same way, cli.py:120-122)
        t0 = time.perf_counter()
        ref = StateVector(n, dtype=np.complex128, device=args.device)
        for g in to_gates(circuit):
            ref.apply(g)
        expected = ref.logical_amplitudes()
        timings["verify_s"] = time.perf_counter() - t0
        err = float(np.abs(a64 - expected).max())
        tol = 1e-5 if dtype == np.complex64 else 1e-10
        verification = {"passed": bool(err <= tol), "max_error": err}

    report = make_report("simulate", engine=args.engine, params=params, counters=counters, digest=digest,
                         verification=verification)
    # device times and achieved bandwidth vary run to run: keep them with the timings
    timings["kernels"] = counters.pop("kernels")
    timings["hbm_GB_per_s"] = counters.pop("hbm_GB_per_s")
    report["timings"] = timings
    report["timings"]["wall_s"] = time.perf_counter() - t_start
    emit(report, args.out)
    if verification is not None and not verification["passed"]:
        return EXIT_VERIFY
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="duetsim-b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    sim = sub.add_parser("simulate", help="run a circuit on the state-vector engine")
    sim.add_argument("--seed", type=int, default=0)
    sim.add_argument("--out", help="also write the JSON report here")
    sim.add_argument("--circuit", choices=["qft", "qv", "qaoa"])
    sim.add_argument("--circuit-file")
    sim.add_argument("--n", type=int, default=4)
    sim.add_argument("--depth", type=int, default=30)
    sim.add_argument("--p", type=int, default=2)
    sim.add_argument("--engine", choices=["sv", "sv-dist", "mps", "tn"], default="sv")
    sim.add_argument("--global-bits", type=int, default=1)
    sim.add_argument("--workers", type=int, default=default_workers())
    sim.add_argument("--max-fused-gate-size", type=int, default=None)
    sim.add_argument("--max-fused-diagonal-gate-size", type=int, default=None)
    sim.add_argument("--fusion", default=None,
                     help="fold:K (phase-folding fuser), cluster:K (cluster-merging fuser) or auto:K (fewer passes of the two)")
    sim.add_argument("--dtype", choices=sorted(DTYPES), default="c128")
    sim.add_argument("--device", type=int, default=None)
    sim.add_argument("--gpus", type=int, default=1, help="shard the state over N GPUs (one host process)")
    sim.add_argument("--verify", action="store_true")
    sim.add_argument("--dry-run", action="store_true")
    sim.set_defaults(func=cmd_simulate)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except InvalidArgumentError as e:
        print(json.dumps({"error": "invalid-argument", "detail": str(e)}), file=sys.stderr)
        return EXIT_VERIFY


if __name__ == "__main__":
    sys.exit(main())
