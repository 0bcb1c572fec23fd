#!/bin/bash
for S in 0 1; do echo "split=$S"; OZ2_MOD_SPLIT=$S timeout 300 python bench.py --size 4096 --steps 20 --warmup 5 --no-extras | grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}'; done > gpurun_out/split_bench.log 2>&1
for S in 0 1; do echo "split=$S"; OZ2_MOD_SPLIT=$S timeout 300 python tools/shape_probe.py 4096 4096 65536 13; OZ2_MOD_SPLIT=$S timeout 300 python tools/shape_probe.py 2048 2048 16384 13; OZ2_MOD_SPLIT=$S timeout 300 python tools/shape_probe.py 1024 1024 16384 13; done >> gpurun_out/split_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests3.log
echo done
