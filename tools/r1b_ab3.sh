#!/bin/bash
{ timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 8;
  timeout 900 python tools/ab_probe.py 32768 13 OZ2_FUSED_CRT 1 0 3; } > gpurun_out/ab_fused3.log 2>&1
OZ2_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --size 4096 > gpurun_out/bench_2rank_gloo.log 2>&1; echo rc=$? >> gpurun_out/bench_2rank_gloo.log
echo done
