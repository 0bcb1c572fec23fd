#!/bin/bash
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
OZ2_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --n 4096 > gpurun_out/bench_2rank_gloo.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
