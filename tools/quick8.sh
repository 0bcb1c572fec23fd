#!/bin/bash
# full GPU suite (incl. blocking) + phases
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_parity_blocking_gpu.py tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 200 python tools/profile_once.py 16384 13 4 > gpurun_out/phases.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum --clock-control none -k regex:k_digits --csv python tools/profile_once.py 16384 13 1 > gpurun_out/dig_ncu.csv 2>&1
echo done
