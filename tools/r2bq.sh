# round 2 session 4: fused CRT below k = 16384 with the round-2 epilogue (auto = separate k_crt)
mkdir -p gpurun_out
o=gpurun_out/r2bq_ab.log; : > $o
timeout 400 python tools/ab_multi.py 8192 13 "fused_crt=1" "-" 8 >> $o 2>&1
timeout 400 python tools/ab_multi.py 12288 13 "fused_crt=1" "-" 6 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 "fused_crt=1" "-" 4 8192 >> $o 2>&1
timeout 400 python tools/ab_multi.py 8192 20 "fused_crt=1" "-" 8 >> $o 2>&1
echo done >> $o
