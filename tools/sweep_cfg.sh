#!/bin/bash
# residue-GEMM configuration sweep at 16384^3 N=13: CTA group x throttle (lead, chunk)
for CG in 1 2; do
 for LC in "0 16" "1 0" "2 16" "4 16" "2 8" "8 8"; do
  set -- $LC
  echo "cg=$CG lead=$1 chunk=$2"
  OZ2_CG=$CG OZ2_SYNC_LEAD=$1 OZ2_SYNC_CHUNK=$2 timeout 120 python tools/profile_once.py 16384 13 3 | tail -1
 done
done
