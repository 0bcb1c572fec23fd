#!/bin/bash
timeout 300 python bench.py --size 4096 --steps 20 --warmup 5 --no-extras | grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' > gpurun_out/crt_bench.log 2>&1
OZ2_FUSED_CRT=0 timeout 300 python tools/profile_once.py 16384 13 3 >> gpurun_out/crt_bench.log 2>&1
timeout 300 python tools/shape_probe.py 1024 1024 16384 13 >> gpurun_out/crt_bench.log 2>&1
timeout 300 python tools/shape_probe.py 2048 2048 16384 13 >> gpurun_out/crt_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests4.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests4.log
echo done
