timeout 600 python -m pytest tests/test_fusion_fold.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for f in fold4 fold5 fold3 5,6; do timeout 300 python tools/profile_step.py --n 33 --fusion $f --steps 1 --timed 2 2>&1 | head -1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches33_fold5.csv python tools/profile_step.py --n 33 --fusion fold5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches33_fold4.csv python tools/profile_step.py --n 33 --fusion fold4 > /dev/null 2>&1
