timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -c 2500 gpurun_out/bench7.json; tail -3 gpurun_out/bench7.err
DSV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench7_2rank.json 2> gpurun_out/bench7_2rank.err; tail -c 1500 gpurun_out/bench7_2rank.json; tail -5 gpurun_out/bench7_2rank.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench7_ref.json 2>&1; tail -c 800 gpurun_out/bench7_ref.json
