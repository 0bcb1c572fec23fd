#!/bin/bash
{ OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 13 OZ2_CRT_GENERIC 0 1 6;
  OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 15 OZ2_CRT_GENERIC 0 1 6 16384 int8;
  timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 6; } > gpurun_out/ab_crt5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_crt" -c 1 -o /tmp/crt_src python tools/profile_once.py 16384 15 1 int8 > gpurun_out/ncu_crt.log 2>&1
ncu -i /tmp/crt_src.ncu-rep --page source --csv --print-source sass > gpurun_out/crt_src.csv 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_int8_gpu.py -m gpu -q -x > gpurun_out/gpu_tests10.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests10.log
echo done
