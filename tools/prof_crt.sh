#!/bin/bash
OZ2_FUSED_CRT=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_crt" -c 1 -o gpurun_out/prof_crt16k python tools/profile_once.py 16384 13 1 > gpurun_out/prof_crt.log 2>&1
for F in 0 1; do
OZ2_FUSED_CRT=$F timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/gemm16k_fused$F.csv 2>&1
done
echo done
