#!/bin/bash
{ OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 13 OZ2_CRT_GENERIC 0 1 6;
  OZ2_FUSED_CRT=0 timeout 600 python tools/ab_probe.py 16384 15 OZ2_CRT_GENERIC 0 1 6 16384 int8; } > gpurun_out/ab_crt4.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_int8_gpu.py tests/test_parity_karatsuba_gpu.py -m gpu -q -x > gpurun_out/gpu_tests8.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests8.log
echo done
