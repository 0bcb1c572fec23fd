#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_int8_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "int8 or depth or cg2" > gpurun_out/int8_tests.log 2>&1; echo rc=$? >> gpurun_out/int8_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --scheme int8 --moduli 14 --steps 5 --warmup 3 --no-extras > gpurun_out/bench_int8.log 2>&1
echo done
