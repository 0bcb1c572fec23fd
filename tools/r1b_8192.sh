#!/bin/bash
run() { echo "$1"; env $1 timeout 300 python bench.py --size 8192 --steps 60 --warmup 5 --no-extras | grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"clocks": {[^}]*}'; }
{ run "X=0"; run "OZ2_MOD_SPLIT=1"; run "OZ2_FUSED_CRT=0"; run "OZ2_SYNC_LEAD=0"; run "OZ2_SYNC_CHUNK=4"; run "OZ2_CG=1"; run "X=0"; } > gpurun_out/b8192.log 2>&1
echo done
