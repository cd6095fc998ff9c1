"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's state-vector hot path
(/root/reference/pkg/src/duetsim/statevec.py, core.py) used as the checker
for the CUDA engine.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; the product path
(paper_2308_01999_b200) never does and has no CPU fallback.

Parity pinning: the restatement is checked against golden vectors produced
by running the reference package itself in the build container
(oracle/gen_golden.py -> tests/golden/), see tests/test_oracle_golden.py.
The reference's arithmetic lives in NumPy (numpy>=1.24, pkg/pyproject.toml:11;
generated with numpy 2.3.5 / scipy-openblas 0.3.30): complex products use
NumPy's FMA form re = fma(dr, ar, -(di*ai)), im = fma(dr, ai, di*ar), dense
gates go through BLAS c/zgemm.
"""
