#!/bin/bash
# tests + phases for both GEMM variants at 16384^3 N=13
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for CG in 1 2; do echo "cg=$CG"; OZ2_CG=$CG timeout 120 python tools/profile_once.py 16384 13 3 | tail -2; done > gpurun_out/phases.log 2>&1
OZ2_CG=2 timeout 300 ncu --set full --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 -o gpurun_out/prof_cg2b python tools/profile_once.py 8192 13 1 > gpurun_out/prof_cg2b.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum -k regex:"k_crt" -c 1 --csv python tools/profile_once.py 8192 13 1 > gpurun_out/crt.csv 2>&1
