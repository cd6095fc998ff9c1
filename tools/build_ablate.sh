#!/bin/bash
# Ablation builds of tc.cu (diagnostics only, never the product): each variant
# removes one stage so its cost shows in tools/tc_bench.py.
#   DSV_LIBRARY=paper_2308_01999_b200/_ablate/<v>/libdsv.so python tools/tc_bench.py ...
set -e
cd "$(dirname "$0")/.."
B=paper_2308_01999_b200
for v in NOPHASE NOSPLIT NOEPI NOMMA; do
  mkdir -p $B/_ablate/$v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude \
    -DDSV_AB_$v -c $B/csrc/tc.cu -o $B/_ablate/$v/tc.o
  objs=$(ls $B/_build/*.o | grep -v '/tc.o$')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $B/_ablate/$v/libdsv.so $objs $B/_ablate/$v/tc.o -lcudart
done
