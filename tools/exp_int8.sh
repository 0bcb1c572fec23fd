#!/bin/bash
mkdir -p gpurun_out
for cfg in "" "OZ2_SYNC_LEAD=0" "OZ2_FUSED_CRT=0" "OZ2_SYNC_LEAD=2" "OZ2_SYNC_CHUNK=32" "OZ2_CG=1"; do
  echo "== $cfg" >> gpurun_out/exp_int8.log
  env $cfg timeout 120 python tools/profile_once.py 16384 14 3 int8 >> gpurun_out/exp_int8.log 2>&1
done
echo done
