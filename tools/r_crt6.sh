#!/bin/bash
{ OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 13 OZ2_CRT_GENERIC 0 1 6;
  OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 15 OZ2_CRT_GENERIC 0 1 6 16384 int8;
  timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 6;
  timeout 600 python tools/ab_probe.py 8192 13 OZ2_FUSED_CRT 1 0 12; } > gpurun_out/ab_crt6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_crt" -c 1 --csv python tools/profile_once.py 16384 15 1 int8 > gpurun_out/ncu_crt6.csv 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests11.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests11.log
echo done
