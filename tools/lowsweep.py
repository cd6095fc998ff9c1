import sys, json; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2308_01999_b200 import gates as G
from paper_2308_01999_b200.statevec import StateVector
from tools.tc_bench import time_op
from tools.sweep import peak
n=int(sys.argv[1]); pk=peak()
sv=StateVector(n, dtype=np.complex64); rng=np.random.default_rng(0)
for tg in [(1,),(0,1),(1,2),(2,3),(0,1,2),(1,2,3),(2,3,4),(3,4,5),(1,3),(0,2),(1,2,4),(0,3,5),(10,11,12)]:
    g=G.DenseGate(G.random_unitary(1<<len(tg), rng), tg)
    ms,b=time_op(sv,g)
    print(tg, f"{b/ms/1e6:.0f} GB/s  {b/ms/1e6/pk:.2f}")
for tg in [(0,1),(1,2),(0,1,2),(1,2,3),(4,5)]:
    k=len(tg); perm=rng.permutation(1<<k); d=np.exp(1j*rng.uniform(0,6.3,1<<k))
    ms,b=time_op(sv,G.PermutationGate(perm,d,tg))
    print("perm",tg, f"{b/ms/1e6:.0f} GB/s  {b/ms/1e6/pk:.2f}")
for pairs in ([(0, n-1)], [(3, 20)], [(0,1),(5,n-2)]):
    nat=sv.native; import statistics
    ts=[]
    for _ in range(4):
        nat.prof_reset(); nat.prof_enable(True); sv.swap_index_bits(pairs); pr=nat.prof_read(); nat.prof_enable(False)
        ts.append(sum(v['ms'] for v in pr.values())); b=sum(v['bytes'] for v in pr.values())
    ms=statistics.median(ts); print("swap",pairs, f"{b/ms/1e6:.0f} GB/s  {b/ms/1e6/pk:.2f}")
