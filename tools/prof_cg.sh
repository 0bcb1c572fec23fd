#!/bin/bash
for CG in 1 2; do
  OZ2_CG=$CG timeout 300 ncu --set full --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 -o gpurun_out/prof_cg$CG python tools/profile_once.py 8192 13 1 > gpurun_out/prof_cg$CG.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:"k_digits|k_crt" -c 3 -o gpurun_out/prof_prep8k_v2 python tools/profile_once.py 8192 13 1 > gpurun_out/ncu_prep2.log 2>&1
OZ2_CG=1 timeout 120 python tools/profile_once.py 16384 13 3 > gpurun_out/phases16k_v2.log 2>&1
