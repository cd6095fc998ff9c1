timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile or dense or golden_single" 2>&1 | tail -3
timeout 600 python tools/sweep.py --n 30 --what targets > gpurun_out/sweep30d.json 2> gpurun_out/sweep30d.err; tail -3 gpurun_out/sweep30d.err
DSV_DISABLE_TILE=1 timeout 600 python tools/sweep.py --n 30 --what targets > gpurun_out/sweep30d_notile.json 2> gpurun_out/sweep30d_notile.err
