#!/usr/bin/env python
"""Large seeded fuzz of the B200 engine against the CPU oracle (a longer run
of tests/test_gpu_fuzz.py's single-gate cases): random sizes 1..20, both
dtypes, dense / diagonal / generalised-permutation gates of arity 1..7 with
up to 2 controls, random states.  Permutations and diagonals must be
bit-exact, dense gates within the north_star bars (conftest).

    python tools/fuzz_big.py 3000 > profiles/fuzz_r2_big.txt
    python tools/fuzz_big.py 400 circuits   # fused circuits (fold / cluster, k = 3..6)
    python tools/fuzz_big.py 300 shards     # sharded engine, P = 2..8 segments
"""
import sys
import time
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

from conftest import assert_state_close, random_state  # noqa: E402
from oracle import sv_oracle as O  # noqa: E402
from paper_2308_01999_b200 import _native as N  # noqa: E402
from paper_2308_01999_b200 import gates as G  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    rng = np.random.default_rng(20261017)
    kinds, classes, fails = Counter(), Counter(), []
    t0 = time.time()
    for c in range(cases):
        n = int(rng.integers(1, 21))
        dtype = (np.complex64, np.complex128)[int(rng.integers(0, 2))]
        k = int(rng.integers(1, min(7, n) + 1))
        qs = [int(q) for q in rng.permutation(n)]
        targets = tuple(qs[:k])
        nc = int(rng.integers(0, min(2, n - k) + 1))
        ctrls = tuple((qs[k + i], int(rng.integers(0, 2))) for i in range(nc))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            g = G.DenseGate(G.random_unitary(1 << k, rng), targets, ctrls)
        else:
            perm = np.arange(1 << k) if kind == 1 else rng.permutation(1 << k)
            g = G.PermutationGate(perm, np.exp(1j * rng.uniform(0, 6.3, 1 << k)), targets, ctrls)
        st = random_state(n, rng, dtype)
        sv = StateVector.from_amplitudes(st)
        nat = sv.native
        nat.prof_reset()
        nat.prof_enable(True)
        sv.apply(g)
        for cl in nat.prof_read():
            classes[cl] += 1
        nat.prof_enable(False)
        kinds[("dense", "diag", "perm")[kind], np.dtype(dtype).name, k] += 1
        try:
            if kind == 0:
                ref = st.astype(np.complex128)
                O.apply_gate(ref, n, G.DenseGate(np.asarray(g.matrix, dtype=dtype).astype(np.complex128), g.targets,
                                                 g.controls, unitary=False))
                assert_state_close(sv.amplitudes, ref, dtype)
            else:
                want = st.copy()
                O.apply_gate(want, n, g)
                np.testing.assert_array_equal(sv.amplitudes, want)
        except AssertionError as e:
            fails.append((c, n, np.dtype(dtype).name, kind, targets, ctrls, str(e)[:200]))
    print(f"fuzz: {cases} cases in {time.time() - t0:.0f} s, {len(fails)} failures")
    print("kernel classes hit:", dict(sorted(classes.items())))
    print("gate kinds:", len(kinds), "distinct (kind, dtype, arity) combinations")
    for f in fails[:20]:
        print("FAIL", f)
    sys.exit(1 if fails else 0)


def circuits():
    """Random circuits and QFTs through the fold and cluster fusers (phased
    windows on every tensor-core kernel) against the unfused oracle."""
    from paper_2308_01999_b200.circuits import gen_qft, gen_qv, random_gate_sequence, to_gates
    from paper_2308_01999_b200.fusion_cluster import fuse_cluster
    from paper_2308_01999_b200.fusion_fold import fuse_fold

    cases = int(sys.argv[1])
    rng = np.random.default_rng(20261018)
    classes, fails = Counter(), []
    t0 = time.time()
    for c in range(cases):
        n = int(rng.integers(8, 19))
        dtype = (np.complex64, np.complex128)[c % 2]
        which = int(rng.integers(0, 3))
        gates = (random_gate_sequence(n, 40, rng, max_arity=3) if which == 0 else
                 to_gates(gen_qft(n)) if which == 1 else to_gates(gen_qv(n, 4, seed=int(rng.integers(0, 1 << 30)))))
        k = int(rng.integers(3, 7))
        fuser = (fuse_fold, fuse_cluster)[int(rng.integers(0, 2))]
        ops = fuser(gates, k).ops
        st = random_state(n, rng, dtype)
        sv = StateVector.from_amplitudes(st)
        nat = sv.native
        nat.prof_reset()
        nat.prof_enable(True)
        for op in ops:
            sv.apply(op)
        for cl in nat.prof_read():
            classes[cl] += 1
        nat.prof_enable(False)
        want = O.run_circuit(gates, n, state=st.astype(np.complex128))
        try:
            assert_state_close(sv.logical_amplitudes(), want, dtype)
        except AssertionError as e:
            fails.append((c, n, np.dtype(dtype).name, which, k, fuser.__name__, str(e)[:200]))
    print(f"circuit fuzz: {cases} circuits in {time.time() - t0:.0f} s, {len(fails)} failures")
    print("kernel classes hit:", dict(sorted(classes.items())))
    for f in fails[:20]:
        print("FAIL", f)
    sys.exit(1 if fails else 0)


def shards():
    """Random circuits on the sharded engine (P = 2, 4, 8 segments on one
    device: the multi-GPU exchange and relocation logic) against the oracle;
    permutation-only circuits must match the unsharded engine bit for bit."""
    from paper_2308_01999_b200.circuits import gen_qft, random_gate_sequence, to_gates
    from paper_2308_01999_b200.shard import ShardedStateVector

    cases = int(sys.argv[1])
    rng = np.random.default_rng(20261019)
    fails = []
    t0 = time.time()
    for c in range(cases):
        n = int(rng.integers(6, 17))
        dtype = (np.complex64, np.complex128)[c % 2]
        P = int(2 ** rng.integers(1, 4))
        gates = random_gate_sequence(n, 30, rng, max_arity=3) if c % 3 else to_gates(gen_qft(n))
        sh = ShardedStateVector(n, [0] * P, dtype)
        sh.run(gates)
        got = sh.gather_logical()
        sh.close()
        want = O.run_circuit(gates, n)
        try:
            assert_state_close(got, want, dtype)
        except AssertionError as e:
            fails.append((c, n, np.dtype(dtype).name, P, str(e)[:200]))
    print(f"shard fuzz: {cases} circuits in {time.time() - t0:.0f} s, {len(fails)} failures")
    for f in fails[:20]:
        print("FAIL", f)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "circuits":
        circuits()
    elif len(sys.argv) > 2 and sys.argv[2] == "shards":
        shards()
    else:
        main()
