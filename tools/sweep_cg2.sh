#!/bin/bash
for LC in "0 16" "2 16" "4 16" "2 4" "4 4" "8 4"; do
  set -- $LC
  echo "cg=2 lead=$1 chunk=$2"
  OZ2_CG=2 OZ2_SYNC_LEAD=$1 OZ2_SYNC_CHUNK=$2 timeout 120 python tools/profile_once.py 16384 13 3 | tail -1
done
