#!/bin/bash
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
run() { echo "== $*"; env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 2>&1 | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' '; echo; }
for LC in "1 8" "1 6" "1 10" "1 12" "2 6" "3 4" "4 2" "1 16"; do set -- $LC; run OZ2_SYNC_LEAD=$1 OZ2_SYNC_CHUNK=$2; done
