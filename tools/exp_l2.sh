#!/bin/bash
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
run() { echo "== $*"; env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 2>&1 | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}'; }
run OZ2_L2PROMO=3
run OZ2_L2PROMO=0
run OZ2_L2PROMO=2
run OZ2_SYNC_LEAD=1 OZ2_SYNC_CHUNK=8
run OZ2_SYNC_LEAD=2 OZ2_SYNC_CHUNK=4
run OZ2_SYNC_LEAD=0
