#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
OZ2_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --size 4096 > gpurun_out/bench_2rank_gloo.log 2>&1
timeout 200 python tools/profile_once.py 16384 13 3 > gpurun_out/phases.log 2>&1
echo done
