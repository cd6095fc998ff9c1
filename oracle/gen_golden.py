"""Generate tests/golden/*.pkl.gz by running the REFERENCE package itself.

TEST INFRASTRUCTURE.  Run in the build container, where the read-only
reference is mounted:

    python oracle/gen_golden.py            # writes tests/golden/

It imports ``duetsim`` from /root/reference/pkg/src (the unmodified reference,
numpy-only) and records inputs + outputs of the state-vector hot path.  The
fixtures pin both the oracle restatement (tests/test_oracle_golden.py) and the
CUDA engine (tests/test_gpu_parity.py).  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import gzip
import os
import pickle
import sys
from pathlib import Path

REF_SRC = Path(os.environ.get("DUETSIM_REF_SRC", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
for k in ("OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "OMP_NUM_THREADS"):
    os.environ.setdefault(k, "1")

import numpy as np  # noqa: E402

import duetsim  # noqa: E402
from duetsim import gates as G  # noqa: E402
from duetsim.circuits import gen_qft, gen_qv, to_gates  # noqa: E402
from duetsim.core import bit_permute  # noqa: E402
from duetsim.distsim import SegmentedStateVector  # noqa: E402
from duetsim.fusion import FusionConfig, fuse  # noqa: E402
from duetsim.statevec import StateVector, run_circuit_sv  # noqa: E402

assert str(REF_SRC) in duetsim.__file__, f"not the reference package: {duetsim.__file__}"


def gate_spec(g) -> dict:
    if isinstance(g, G.PermutationGate):
        return {"kind": "perm", "perm": g.permutation.copy(), "diag": g.diagonal.copy(),
                "targets": tuple(g.targets), "controls": tuple(g.controls)}
    return {"kind": "dense", "matrix": g.matrix.copy(), "targets": tuple(g.targets),
            "controls": tuple(g.controls), "unitary": bool(g.unitary)}


def random_state(n, rng):
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)


def random_gate(n, rng, max_arity=3, max_ctrl=2):
    k = int(rng.integers(1, min(max_arity, n) + 1))
    qs = rng.choice(n, size=min(n, k + max_ctrl), replace=False).tolist()
    targets = tuple(int(q) for q in qs[:k])
    nc = int(rng.integers(0, min(max_ctrl, n - k) + 1))
    controls = tuple((int(q), int(rng.integers(0, 2))) for q in qs[k:k + nc])
    kind = int(rng.integers(0, 3))
    dim = 1 << k
    if kind == 0:
        return G.DenseGate(G.random_unitary(dim, rng), targets, controls)
    ph = np.exp(1j * rng.uniform(0, 2 * np.pi, dim))
    if kind == 1:
        # some entries exactly 1 so the engine's skip path is exercised
        ph[rng.random(dim) < 0.3] = 1.0
        return G.PermutationGate(np.arange(dim), ph, targets, controls)
    return G.PermutationGate(rng.permutation(dim), ph, targets, controls)


def fam_sv_random(rng):
    cases = []
    for i in range(48):
        n = int(rng.integers(2, 10))
        count = int(rng.integers(5, 31))
        gates = [random_gate(n, rng) for _ in range(count)]
        for dt in (np.complex128, np.complex64):
            sv = StateVector(n, dtype=dt)
            for g in gates:
                sv.apply(g)
            cases.append({"n": n, "dtype": np.dtype(dt).name, "gates": [gate_spec(g) for g in gates],
                          "out": sv.amplitudes.copy()})
    return cases


def fam_single_ops(rng):
    """One gate on a random state: inputs + exact outputs (bit-exact checks)."""
    cases = []
    for i in range(160):
        n = int(rng.integers(3, 11))
        g = random_gate(n, rng, max_arity=min(6, n), max_ctrl=2)
        for dt in (np.complex128, np.complex64):
            st = random_state(n, rng).astype(dt)
            sv = StateVector.from_amplitudes(st.copy())
            sv.apply(g)
            cases.append({"n": n, "dtype": np.dtype(dt).name, "gate": gate_spec(g), "in": st,
                          "out": sv.amplitudes.copy()})
    return cases


def fam_swap_access(rng):
    cases = []
    for i in range(40):
        n = int(rng.integers(2, 11))
        dt = np.complex128 if i % 2 else np.complex64
        st = random_state(n, rng).astype(dt)
        bits = rng.permutation(n).tolist()
        npairs = int(rng.integers(1, n // 2 + 1))
        pairs = [(int(bits[2 * p]), int(bits[2 * p + 1])) for p in range(npairs)]
        sv = StateVector.from_amplitudes(st.copy())
        sv.swap_index_bits(pairs)
        ordering = rng.permutation(n).tolist()
        begin = int(rng.integers(0, 1 << (n - 1)))
        end = int(rng.integers(begin + 1, (1 << n) + 1))
        acc = sv.access(ordering, begin, end)
        logical = sv.logical_amplitudes()
        vals = (rng.standard_normal(end - begin) + 1j * rng.standard_normal(end - begin)).astype(dt)
        sv2 = StateVector.from_amplitudes(st.copy())
        sv2.access_set(ordering, begin, vals)
        cases.append({"n": n, "dtype": np.dtype(dt).name, "in": st, "pairs": pairs,
                      "out": sv.amplitudes.copy(), "bit_map": list(sv.bit_map),
                      "ordering": ordering, "begin": begin, "end": end, "access": acc,
                      "logical": logical, "set_values": vals, "after_set": sv2.amplitudes.copy()})
    return cases


def fam_measure(rng):
    cases = []
    for i in range(40):
        n = int(rng.integers(2, 10))
        dt = np.complex128 if i % 2 else np.complex64
        st = random_state(n, rng).astype(dt)
        k = int(rng.integers(1, min(4, n) + 1))
        qubits = rng.choice(n, size=k, replace=False).tolist()
        r = float(rng.random())
        sv = StateVector.from_amplitudes(st.copy())
        probs = sv.probabilities(qubits)
        outcome = sv.measure(qubits, r, collapse=True)
        # expectation: random Pauli list + dense hermitian
        paulis = []
        for _ in range(3):
            m = int(rng.integers(1, min(4, n) + 1))
            qs = rng.choice(n, size=m, replace=False).tolist()
            fac = tuple((int(q), str(rng.choice(list("IXYZ")))) for q in qs)
            coef = complex(rng.standard_normal(), rng.standard_normal()) if rng.random() < 0.5 else 1.0
            paulis.append(G.PauliString(fac, coef))
        sv3 = StateVector.from_amplitudes(st.copy())
        ev_pauli = sv3.expectation(paulis)
        kd = int(rng.integers(1, min(3, n) + 1))
        tq = tuple(int(q) for q in rng.choice(n, size=kd, replace=False))
        a = rng.standard_normal((1 << kd, 1 << kd)) + 1j * rng.standard_normal((1 << kd, 1 << kd))
        herm = (a + a.conj().T) / 2
        ev_dense = sv3.expectation(G.DenseGate(herm, tq, unitary=False))
        # rotation
        theta = float(rng.uniform(0, 2 * np.pi))
        rot = paulis[0]
        rot_nontrivial = G.PauliString(tuple(f for f in rot.factors) or ((0, "Z"),), rot.coefficient)
        sv4 = StateVector.from_amplitudes(st.copy())
        sv4.apply_pauli_rotation(theta, rot_nontrivial)
        # sampling (physical outcomes pinned through bitstrings)
        seed = int(rng.integers(0, 1000))
        order = rng.permutation(n).tolist() if i % 3 == 0 else None
        shots = sv3.sample(257, qubit_order=order, seed=seed)
        cases.append({
            "n": n, "dtype": np.dtype(dt).name, "in": st, "qubits": qubits, "r": r,
            "probs": probs, "outcome": outcome, "collapsed": sv.amplitudes.copy(),
            "paulis": [(p.factors, complex(p.coefficient)) for p in paulis], "ev_pauli": complex(ev_pauli),
            "herm": herm, "herm_targets": tq, "ev_dense": complex(ev_dense),
            "theta": theta, "rot": (rot_nontrivial.factors, complex(rot_nontrivial.coefficient)),
            "rotated": sv4.amplitudes.copy(), "seed": seed, "order": order, "shots": shots,
            "norm": sv3.norm_squared(),
        })
    return cases


def fam_fusion(rng):
    cases = []
    circs = []
    for n in (3, 5, 8):
        circs.append(("qft", n, to_gates(gen_qft(n))))
    circs.append(("qv", 6, to_gates(gen_qv(6, 5, seed=3))))
    for i in range(12):
        n = int(rng.integers(3, 8))
        circs.append(("rand", n, [random_gate(n, rng, max_arity=2, max_ctrl=1) for _ in range(int(rng.integers(5, 40)))]))
    for name, n, gates in circs:
        for cfg in ((2, 3), (3, 4), (4, 6), (5, 6)):
            fc = fuse(gates, FusionConfig(*cfg))
            passthrough = [any(fg is g for g in gates) for fg in fc.gates]
            cases.append({
                "name": name, "n": n, "cfg": cfg, "gates": [gate_spec(g) for g in gates],
                "fused": [gate_spec(g) for g in fc.gates], "provenance": fc.provenance,
                "passthrough": passthrough,
                "out": run_circuit_sv(fc.gates, n).amplitudes.copy(),
            })
    counts = {}
    for (k, d) in ((2, 6), (3, 6), (4, 6), (5, 6), (5, 5), (5, 10), (4, 4)):
        counts[f"qft33_{k}_{d}"] = len(fuse(to_gates(gen_qft(33)), FusionConfig(k, d)))
    counts["qv33_5_6"] = len(fuse(to_gates(gen_qv(33, 30, seed=0)), FusionConfig(5, 6)))
    counts["qv34_5_6"] = len(fuse(to_gates(gen_qv(34, 30, seed=0)), FusionConfig(5, 6)))
    counts["qv34_4_6"] = len(fuse(to_gates(gen_qv(34, 30, seed=0)), FusionConfig(4, 6)))
    counts["qft20_5_6"] = len(fuse(to_gates(gen_qft(20)), FusionConfig(5, 6)))
    return {"cases": cases, "counts": counts}


def fam_distsim(rng):
    cases = []
    for i in range(30):
        n = int(rng.integers(4, 9))
        g = int(rng.integers(1, min(3, n - 2) + 1))
        workers = int(rng.choice([1, 2, 4]))
        if i % 3 == 0:
            gates = to_gates(gen_qft(n))
        else:
            gates = [random_gate(n, rng, max_arity=2, max_ctrl=1) for _ in range(int(rng.integers(5, 25)))]
        with SegmentedStateVector(n, g, workers) as ssv:
            ssv.run(gates)
            stats = ssv.transfer_stats().as_dict()
            segs = [s.copy() for s in ssv.segments]
            qmap = list(ssv.qubit_map)
            logical = ssv.to_statevector().amplitudes.copy()
        cases.append({"n": n, "g": g, "workers": workers, "gates": [gate_spec(x) for x in gates],
                      "stats": stats, "segments": segs, "qubit_map": qmap, "logical": logical})
    # explicit index-bit swaps with mixed pair kinds
    swaps = []
    for i in range(30):
        n = int(rng.integers(3, 9))
        g = int(rng.integers(1, min(3, n - 1) + 1))
        workers = int(rng.choice([1, 2, 4]))
        st = random_state(n, rng)
        bits = rng.permutation(n).tolist()
        npairs = int(rng.integers(1, n // 2 + 1))
        pairs = [(int(bits[2 * p]), int(bits[2 * p + 1])) for p in range(npairs)]
        ssv = SegmentedStateVector(n, g, workers)
        L = 1 << (n - g)
        for s in range(1 << g):
            ssv.segments[s][:] = st[s * L:(s + 1) * L]
        ssv.distributed_index_bit_swap(pairs)
        swaps.append({"n": n, "g": g, "workers": workers, "in": st, "pairs": pairs,
                      "segments": [s.copy() for s in ssv.segments], "stats": ssv.stats.as_dict(),
                      "qubit_map": list(ssv.qubit_map)})
        ssv.close()
    return {"runs": cases, "swaps": swaps}


def fam_misc(rng):
    out = {}
    out["qft_states"] = {n: run_circuit_sv(to_gates(gen_qft(n)), n).amplitudes.copy() for n in range(1, 13)}
    out["counts"] = {"qft33": len(gen_qft(33)), "qv33": len(gen_qv(33, 30, seed=0)),
                     "qv34": len(gen_qv(34, 30, seed=0)), "qft20": len(gen_qft(20))}
    out["qv6_targets"] = [tuple(op.targets) for op in gen_qv(6, 5, seed=3).ops]
    xs = rng.integers(0, 1 << 20, size=64).tolist()
    pairs = [(0, 7), (2, 9), (4, 5)]
    out["bit_permute"] = {"x": xs, "pairs": pairs, "y": [bit_permute(int(x), pairs) for x in xs]}
    rng2 = np.random.default_rng(44)
    st = random_state(5, rng2)
    sv = StateVector.from_amplitudes(st)
    sv.swap_index_bits([(1, 3)])
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "s.bin"
        sv.dump(p)
        out["dump"] = {"in": st, "pairs": [(1, 3)], "bytes": p.read_bytes()}
    # the reference test oracle's random circuit generator (tests/oracles.py:208-226)
    sys.path.insert(0, str(REF_SRC.parent / "tests"))
    from oracles import random_gate_sequence  # noqa: E402
    seqs = []
    for seed, n, count, ar in ((0, 6, 20, 3), (1, 8, 30, 2), (42, 6, 20, 3)):
        seq = random_gate_sequence(n, count, np.random.default_rng(seed), max_arity=ar)
        seqs.append({"seed": seed, "n": n, "count": count, "max_arity": ar,
                     "gates": [gate_spec(g) for g in seq],
                     "out": run_circuit_sv(seq, n).amplitudes.copy()})
    out["random_gate_sequence"] = seqs
    return out


def fam_config1(rng):
    """BASELINE configs[0]: QFT-20 complex128 (runs on the reference as-is),
    unfused (220 gates) and fused with FusionConfig(5, 6) (66 ops), from
    |0...0> and from a seeded random state.  The 16 MiB states are not stored
    whole: 8192 seeded amplitude samples, marginals and the norm are."""
    n = 20
    gates = to_gates(gen_qft(n))
    fc = fuse(gates, FusionConfig(5, 6))
    state_seed = 2020
    st = random_state(n, np.random.default_rng(state_seed))
    idx = np.sort(np.random.default_rng(2021).choice(1 << n, size=8192, replace=False))
    out = {"n": n, "state_seed": state_seed, "idx": idx, "gates": len(gates), "fused_ops": len(fc.gates)}
    for tag, start in (("zero", None), ("random", st)):
        for ftag, gl in (("unfused", gates), ("fused", fc.gates)):
            sv = StateVector.from_amplitudes(start) if start is not None else StateVector(n)
            for g in gl:
                sv.apply(g)
            a = sv.logical_amplitudes()
            out[f"{tag}_{ftag}"] = {"samples": a[idx].copy(), "norm": float(np.vdot(a, a).real),
                                    "marginal_0_19_7_13": sv.probabilities([0, 19, 7, 13]).copy()}
    return out


def fam_cli(rng):
    """The reference CLI's `simulate` reports (cli.py:124-244), timings
    dropped: digests, norms, counters and transfer stats that the GPU CLI
    must reproduce for the same arguments."""
    import contextlib
    import io
    import json

    from duetsim.cli import main as ref_main

    runs = [
        ["simulate", "--circuit", "qft", "--n", "10"],
        ["simulate", "--circuit", "qft", "--n", "12", "--max-fused-gate-size", "4",
         "--max-fused-diagonal-gate-size", "6"],
        ["simulate", "--circuit", "qft", "--n", "10", "--engine", "sv-dist", "--global-bits", "2", "--workers", "2"],
        ["simulate", "--circuit", "qv", "--n", "8", "--seed", "5", "--verify"],
        ["simulate", "--circuit", "qaoa", "--n", "6", "--engine", "sv-dist", "--global-bits", "1", "--verify"],
        ["simulate", "--circuit", "qft", "--n", "20", "--verify"],
    ]
    out = []
    for argv in runs:
        buf, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
            code = ref_main(argv)
        rep = json.loads(buf.getvalue()) if buf.getvalue().strip() else None
        if rep is not None:
            rep.pop("timings", None)
        out.append({"argv": argv, "code": code, "report": rep,
                    "stderr": json.loads(err.getvalue()) if err.getvalue().strip() else None})
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    fams = {
        "sv_random": fam_sv_random,
        "single_ops": fam_single_ops,
        "swap_access": fam_swap_access,
        "measure": fam_measure,
        "fusion": fam_fusion,
        "distsim": fam_distsim,
        "misc": fam_misc,
        "config1": fam_config1,
        "cli": fam_cli,
    }
    only = sys.argv[1:]
    for i, (name, fn) in enumerate(fams.items()):
        if only and name not in only:
            continue
        data = fn(np.random.default_rng(20261017 + i))
        meta = {"generator": "oracle/gen_golden.py", "reference": str(REF_SRC),
                "numpy": np.__version__, "family": name}
        with gzip.open(OUT / f"{name}.pkl.gz", "wb") as fh:
            pickle.dump({"meta": meta, "data": data}, fh, protocol=4)
        print(f"wrote {name}: {(OUT / f'{name}.pkl.gz').stat().st_size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
