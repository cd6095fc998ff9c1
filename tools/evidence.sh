#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench line, ncu launch list of
# one QFT-33 step, ncu --set full of the QFT-30 window kernels.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/profile_step.py --n 33 --fusion fold5 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dense_(tc8|lowt)" -c 7 \
  -o gpurun_out/prof_qft30 python tools/prof_qft_ops.py 30 5 > gpurun_out/prof_qft30.log 2>&1
cat gpurun_out/bench.json gpurun_out/launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dense_lowt" -c 1 \
  -o gpurun_out/prof_lowt28 python tools/prof_qft_ops.py 28 5 > gpurun_out/prof_lowt28.log 2>&1
timeout 900 python tools/sweep.py --n 33 --what targets > gpurun_out/sweep_n33.json 2> gpurun_out/sweep_n33.err
timeout 900 python tools/ops_sweep.py > gpurun_out/ops_sweep.json 2> gpurun_out/ops_sweep.err
