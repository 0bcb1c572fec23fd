# round 2: K-concatenated square cross products vs k (the epilogue-bound small-k regime)
mkdir -p gpurun_out
o=gpurun_out/r2ac.log; : > $o
for k in 1024 2048 4096 8192; do
  timeout 300 python tools/ab_multi.py 16384 13 - "kcat=1" 8 $k >> $o 2>&1
done
timeout 300 python tools/ab_multi.py 8192 13 - "kcat=1" 8 1024 >> $o 2>&1
timeout 300 python tools/ab_multi.py 4096 13 - "kcat=1" 8 4096 >> $o 2>&1
echo done >> $o
