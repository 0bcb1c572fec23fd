#!/bin/bash
# INT8 scheme parity first, then the full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_int8_gpu.py -m gpu -q -x > gpurun_out/int8_tests.log 2>&1; echo rc=$? >> gpurun_out/int8_tests.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
echo done
