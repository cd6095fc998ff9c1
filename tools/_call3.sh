timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 400 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -c 600 gpurun_out/bench3.json; tail -5 gpurun_out/bench3.err
timeout 600 python tools/sweep.py --n 30 --what targets > gpurun_out/sweep30b.json 2> gpurun_out/sweep30b.err; tail -3 gpurun_out/sweep30b.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches33b.csv python tools/profile_step.py --n 33 > gpurun_out/ncu1b.log 2>&1; tail -2 gpurun_out/ncu1b.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_diag_stream -s 20 -c 2 -o gpurun_out/prof_diagstream python tools/profile_step.py --n 28 > gpurun_out/ncu2b.log 2>&1; tail -2 gpurun_out/ncu2b.log
