#!/bin/bash
# Round-2 closing evidence on one B200 (run under gpurun): GPU suite, smoke,
# bench line and the reference arm, ncu launch list of one QFT-33 step (+ DRAM
# bytes), ncu --set full of the complex128 tensor-core window, the
# complex128 per-layout probe, BASELINE.md's configs table.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; tail -2 gpurun_out/r2f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; tail -1 gpurun_out/r2f_smoke.log
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python bench.py --impl reference > gpurun_out/r2f_reference.json 2> gpurun_out/r2f_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2f_launches.csv python tools/profile_step.py --n 33 --fusion fold5 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2f_launches.csv > gpurun_out/r2f_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_tc8d -c 1 \
  -o gpurun_out/r2f_tc8d_n28 python tools/tc8d_one.py 28 3,4,5,6,7 > gpurun_out/r2f_tc8d_ncu.log 2>&1
timeout 300 python tools/tc8d_probe.py 32 tc8d 1,0 > gpurun_out/r2f_tc8d_probe.txt 2>&1
timeout 1200 python tools/configs_table.py > gpurun_out/r2f_configs_table.json 2> gpurun_out/r2f_configs_table.err
cat gpurun_out/r2f_launches.txt
python -c "import json;d=json.load(open('gpurun_out/r2f_bench.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks'])"
python -c "import json;d=json.load(open('gpurun_out/r2f_reference.json'));print(d.get('value'),d.get('unit'))"
