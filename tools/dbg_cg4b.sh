#!/bin/bash
r() { echo "== $*"; env "$@" timeout 60 python tools/dbg_cg4.py $N $K 2>&1 | tail -1; }
N=4096 K=8192; r OZ2_CG=4; r OZ2_CG=2
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size"
for CG in 2 4; do echo "== cg=$CG"; OZ2_CG=$CG timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -s 1 -c 1 --csv python tools/profile_once.py 16384 13 1 2>&1 | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' '; echo; done
for CG in 2 4; do echo "== cg=$CG"; OZ2_CG=$CG timeout 200 python tools/profile_once.py 16384 13 4 | tail -2; done
