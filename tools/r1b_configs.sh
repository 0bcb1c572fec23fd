#!/bin/bash
# BASELINE configs 2, 4, 5 (single GPU): accuracy/throughput sweeps and the 32768^3 bench line
timeout 1200 python tools/accuracy_sweep.py --size 8192 --moduli 12,13,14,15,16,17,18,19,20 --phis 0,1,4 --out gpurun_out/accuracy_8192.json > gpurun_out/acc8192.log 2>&1
timeout 1200 python tools/accuracy_sweep.py --size 4096 --k 65536 --moduli 12,13,14 --phis 0,1 --out gpurun_out/accuracy_4096x65536.json > gpurun_out/acc4096.log 2>&1
timeout 600 python bench.py --size 32768 --moduli 13 --steps 3 --warmup 3 --no-extras > gpurun_out/bench_32768.log 2>&1
timeout 600 python bench.py --size 8192 --moduli 13 --steps 10 --warmup 3 --no-extras > gpurun_out/bench_8192.log 2>&1
echo done
