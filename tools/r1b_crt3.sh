#!/bin/bash
{ timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 6;
  timeout 600 python tools/ab_probe.py 16384 15 OZ2_FUSED_CRT 1 0 6 16384 int8;
  timeout 300 python tools/ab_probe.py 8192 13 OZ2_FUSED_CRT 1 0 12; } > gpurun_out/ab_crt3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests7.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests7.log
echo done
