#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for n in 16384 8192; do for F in 1 0; do echo "fused=$F n=$n"; OZ2_FUSED_CRT=$F timeout 120 python tools/profile_once.py $n 13 3 | tail -2; done; done > gpurun_out/phases.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm_kernel|k_crt" -s 1 -c 2 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/gemm16k.csv 2>&1
OZ2_FUSED_CRT=0 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_crt" -c 1 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/crt16k.csv 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
echo done
