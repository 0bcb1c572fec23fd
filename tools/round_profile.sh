#!/bin/bash
# tests, bench, launch list and full ncu captures of the bench workload's kernels
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python tools/profile_once.py 16384 13 3 > gpurun_out/phases.log 2>&1
OZ2_FUSED_CRT=0 timeout 300 python tools/profile_once.py 16384 13 3 > gpurun_out/phases_unfused.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|k_digits|k_cast|k_rowmax" -c 7 -o gpurun_out/prof16k python tools/profile_once.py 16384 13 1 > gpurun_out/ncu_full16k.log 2>&1
echo done
