# round 2: fused vs separate CRT at k = 8192 with the round-2 epilogue; KCAT auto check
mkdir -p gpurun_out
o=gpurun_out/r2ad.log; : > $o
timeout 300 python tools/ab_multi.py 16384 13 - "fused_crt=1" 8 8192 >> $o 2>&1
timeout 300 python tools/ab_multi.py 8192 13 - "fused_crt=1" 8 8192 >> $o 2>&1
timeout 300 python tools/ab_multi.py 16384 15 - "fused_crt=1" 6 16384 >> $o 2>&1
timeout 300 python tools/phase_probe.py 16384 16384 1024 13 10 >> $o 2>&1
echo done >> $o
