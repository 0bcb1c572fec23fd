# round 2: small-k regression hunt at 16384^2 x 1024 (and 4096): HEAD vs ab_old, knob A/Bs
mkdir -p gpurun_out
o=gpurun_out/r2ab.log; : > $o
for d in . ab_old . ab_old; do
  (cd $d && timeout 300 python tools/phase_probe.py 16384 16384 1024 13 10) >> $o 2>&1
done
timeout 300 python tools/ab_multi.py 16384 13 - "sync_chunk=8" 8 1024 >> $o 2>&1
timeout 300 python tools/ab_multi.py 16384 13 - "epi_sleep=0" 8 1024 >> $o 2>&1
timeout 300 python tools/ab_multi.py 16384 13 - "mod_split=0" 8 1024 >> $o 2>&1
timeout 300 python tools/ab_multi.py 16384 13 - "sync_lead=0" 8 1024 >> $o 2>&1
echo done >> $o
