"""Full-size parity of the headline workload (QFT-33 complex64, fold fuser
k = 5, the bench's kernels): QFT|x> = (1/sqrt N) sum_y w^(x y) |y>, so every
amplitude has modulus 2^-16.5 and, after the final relabel swaps, amplitude y
has phase 2 pi x y / N.  Checked on a 2^20-amplitude strided sample downloaded
from the device plus norm and marginals over 4-qubit subsets (device
reductions over all 2^33 amplitudes)."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2308_01999_b200.circuits import gen_qft, to_gates
from paper_2308_01999_b200.fusion_fold import fuse_fold
from paper_2308_01999_b200.statevec import StateVector

n = 33
N = 1 << n
ops = fuse_fold(to_gates(gen_qft(n)), 5).ops
out = {"n": n, "dtype": "complex64", "cases": []}
rng = np.random.default_rng(5)
for x in (0, int(rng.integers(1, N))):
    sv = StateVector(n, dtype=np.complex64)
    sv.native.set_basis(x)
    for g in ops:
        sv.apply(g)
    norm = sv.norm_squared()
    marg_err = 0.0
    for bits in ([0, 1, 2, 3], [29, 30, 31, 32], [0, 11, 22, 32]):
        p = sv.probabilities(bits)
        marg_err = max(marg_err, float(np.abs(p - 1.0 / 16).max()))
    # strided logical sample: y = s * stride + off
    ys = (np.arange(1 << 20, dtype=np.int64) * (N >> 20) + 12345) % N
    amps = np.array([sv.access(list(sv.bit_map), int(y), int(y) + 1)[0] for y in ys[:4096]])
    want = np.exp(2j * np.pi * ((x * ys[:4096]) % N) / N) / np.sqrt(N)
    err = float(np.abs(amps.astype(np.complex128) - want).max() / (1 / np.sqrt(N)))
    case = {"x": x, "norm_minus_1": norm - 1.0, "marginal_max_err": marg_err, "sample_rel_err": err}
    out["cases"].append(case)
    print(json.dumps(case), flush=True)
    del sv
print(json.dumps(out))
