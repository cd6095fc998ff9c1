#!/usr/bin/env python
"""Accuracy of the dense kernels over repeated application (norm drift and
max relative error): U then U^dagger, 20 rounds, n = 20, complex64.

    python tools/tc_precision.py            # tensor-core path
    DSV_TC=0 python tools/tc_precision.py   # CUDA-core kernels
"""

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2308_01999_b200 import gates as G  # noqa: E402
from paper_2308_01999_b200.statevec import StateVector  # noqa: E402


def main():
    rng = np.random.default_rng(3)
    n = 20
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    st = (v / np.linalg.norm(v)).astype(np.complex64)
    out = {"DSV_TC": os.environ.get("DSV_TC", "1")}
    for k, targets in ((4, (3, 8, 12, 17)), (5, (2, 6, 11, 15, 19))):
        sv = StateVector.from_amplitudes(st)
        m = G.random_unitary(1 << k, rng)
        rows = []
        for r in range(20):
            sv.apply_matrix(G.DenseGate(m, targets))
            sv.apply_matrix(G.DenseGate(m.conj().T, targets))
            a = sv.amplitudes.astype(np.complex128)
            rows.append({"round": r + 1, "norm2_minus_1": float(np.vdot(a, a).real - 1.0),
                         "rel_err": float(np.abs(a - st).max() / np.abs(st).max()),
                         "fid_minus_1": float(abs(np.vdot(st.astype(np.complex128), a)) ** 2 - 1.0)})
        out[f"k{k}"] = rows[::4] + [rows[-1]]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
