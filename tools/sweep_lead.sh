#!/bin/bash
# phases at 16384^3 N=13 for several progress-throttle settings
for L in 0 1 2 4; do
  echo "lead=$L"; OZ2_SYNC_LEAD=$L timeout 120 python tools/profile_once.py 16384 13 4 | tail -2
done
