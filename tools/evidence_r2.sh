#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): GPU suite, smoke, bench line,
# ncu launch list of one QFT-33 step (+ DRAM bytes), ncu --set full of the
# QFT-30 window kernels, the QV-33 window A/B.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2e_gputest.log 2>&1; tail -2 gpurun_out/r2e_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; tail -1 gpurun_out/r2e_smoke.log
python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2e_launches.csv python tools/profile_step.py --n 33 --fusion fold5 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2e_launches.csv > gpurun_out/r2e_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dense_(tc8|lowt)" -c 7 \
  -o gpurun_out/r2e_prof_qft30 python tools/prof_qft_ops.py 30 5 > gpurun_out/r2e_prof_qft30.log 2>&1
cat gpurun_out/r2e_launches.txt
python -c "import json;d=json.load(open('gpurun_out/r2e_bench.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['legs'],d['clocks'])"
