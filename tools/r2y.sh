# round 2: confirm the knob candidates with more rounds (16384^3, N = 13)
mkdir -p gpurun_out
o=gpurun_out/r2y_knobs.log; : > $o
timeout 400 python tools/ab_multi.py 16384 13 - "sq_order=0" 12 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 - "sync_chunk=4" 12 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 - "sq_order=0,sync_chunk=4" 12 >> $o 2>&1
timeout 400 python tools/ab_multi.py 8192 13 - "sq_order=0,sync_chunk=4" 12 >> $o 2>&1
timeout 600 python tools/ab_multi.py 32768 13 - "sq_order=0,sync_chunk=4" 2 >> $o 2>&1
echo done >> $o
