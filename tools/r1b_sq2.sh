#!/bin/bash
for O in 0 1; do OZ2_SQ_ORDER=$O timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_kernel -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/sq_order_ncu_$O.csv 2>&1; done
for O in 0 1; do OZ2_SQ_ORDER=$O timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_kernel -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/sq_order_ncu_b$O.csv 2>&1; done
echo done
