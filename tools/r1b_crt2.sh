#!/bin/bash
for r in 1 2; do timeout 300 python bench.py --size 4096 --steps 20 --warmup 5 --no-extras | grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}'; done > gpurun_out/crt_bench2.log 2>&1
timeout 300 python tools/shape_probe.py 1024 1024 16384 13 >> gpurun_out/crt_bench2.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "schedules or ragged or imported" > gpurun_out/gpu_tests5.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests5.log
echo done
