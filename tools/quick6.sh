#!/bin/bash
# fast-mode parity + benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_fast_gpu.py tests/test_parity_large_gpu.py -m gpu -q -x -k "fast" > gpurun_out/fast_tests.log 2>&1; echo rc=$? >> gpurun_out/fast_tests.log
timeout 600 python bench.py --mode fast --steps 5 --warmup 3 --no-extras > gpurun_out/bench_fast.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_acc.log 2>&1
echo done
