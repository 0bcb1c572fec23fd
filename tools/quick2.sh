#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for F in 1 0; do echo "fused=$F"; OZ2_FUSED_CRT=$F timeout 120 python tools/profile_once.py 16384 13 3 | tail -2; done > gpurun_out/phases.log 2>&1
for F in 1 0; do echo "fused=$F n=8192"; OZ2_FUSED_CRT=$F timeout 120 python tools/profile_once.py 8192 13 3 | tail -1; done >> gpurun_out/phases.log 2>&1
