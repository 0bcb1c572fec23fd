# round 2: knob re-tuning on the row-blocked layout + packed epilogue (16384^3, N = 13)
mkdir -p gpurun_out
o=gpurun_out/r2x_knobs.log; : > $o
timeout 300 python tools/ab_probe.py 16384 13 sync_chunk 8 4 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 sync_chunk 8 16 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 sync_lead 1 2 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 l2_promo 3 2 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 kcat 0 1 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 cta_group 2 4 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 epi_sleep 1000 300 6 >> $o 2>&1
timeout 300 python tools/ab_probe.py 16384 13 sq_order 1 0 6 >> $o 2>&1
echo done >> $o
