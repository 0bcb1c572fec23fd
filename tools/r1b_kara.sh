#!/bin/bash
# Karatsuba-family parity, accuracy study at 16384 (4 phis), karatsuba bench
timeout 900 python -m pytest tests/test_parity_karatsuba_gpu.py tests/test_parity_int8_gpu.py -q -x > gpurun_out/kara_tests.log 2>&1; echo rc=$? >> gpurun_out/kara_tests.log
timeout 1200 python tools/accuracy_sweep.py --out gpurun_out/accuracy_16384.json > gpurun_out/accuracy.log 2>&1
timeout 300 python bench.py --scheme karatsuba --no-extras > gpurun_out/bench_kara.log 2>&1
timeout 300 python bench.py --moduli 12 --no-extras > gpurun_out/bench_n12.log 2>&1
echo done
