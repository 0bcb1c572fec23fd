#!/bin/bash
timeout 400 python -m pytest tests/test_parity_gpu.py -q -x -k "cg4" > gpurun_out/cg4_tests.log 2>&1; echo rc=$? >> gpurun_out/cg4_tests.log
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct"
for CG in 2 4; do echo "== cg=$CG"; OZ2_CG=$CG timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 2>&1 | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' '; echo; done > gpurun_out/cg4_perf.log
for CG in 2 4; do echo "== cg=$CG"; OZ2_CG=$CG timeout 200 python tools/profile_once.py 16384 13 4 | tail -2; done >> gpurun_out/cg4_perf.log 2>&1
