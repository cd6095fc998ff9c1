#!/bin/bash
# Build the committed HEAD's libdsv.so into paper_2308_01999_b200/_ablate/head (same-box A/B runs:
# DSV_LIBRARY=paper_2308_01999_b200/_ablate/head/libdsv.so)
set -e
cd "$(dirname "$0")/.."
B=paper_2308_01999_b200
rm -rf /tmp/headsrc && mkdir -p /tmp/headsrc $B/_ablate/head && rm -f $B/_ablate/head/*.o
git archive HEAD $B/csrc include | tar -x -C /tmp/headsrc
for f in /tmp/headsrc/$B/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I/tmp/headsrc/include -c $f -o $B/_ablate/head/$(basename $f .cu).o 2>/dev/null &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $B/_ablate/head/libdsv.so $B/_ablate/head/*.o -lcudart
echo built $B/_ablate/head/libdsv.so
