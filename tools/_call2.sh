set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "diag or golden_single or large" 2>&1 | tail -5
timeout 400 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -c 1500 gpurun_out/bench2.json
timeout 600 python tools/sweep.py --n 30 > gpurun_out/sweep30.json 2> gpurun_out/sweep30.err; tail -3 gpurun_out/sweep30.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches33.csv python tools/profile_step.py --n 33 > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_diag -s 20 -c 2 -o gpurun_out/prof_diag python tools/profile_step.py --n 28 > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu2.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_dense -s 3 -c 2 -o gpurun_out/prof_dense python tools/profile_step.py --n 28 > gpurun_out/ncu3.log 2>&1; tail -3 gpurun_out/ncu3.log
ls -la gpurun_out
