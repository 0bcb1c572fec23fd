# round 2 session 4: fused CRT with all residue loads issued first (crt_element_prefetch):
# fused-path parity tests, in-step A/B against ab_base, fused-vs-separate below k = 16384
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_large_gpu.py tests/test_parity_int8_gpu.py -m gpu -q -x > gpurun_out/r2br_tests.log 2>&1; echo rc=$? >> gpurun_out/r2br_tests.log
for i in 1 2; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2br_ab_${i}_$(basename $d).log 2>&1
  done
done
o=gpurun_out/r2br_fused.log; : > $o
timeout 400 python tools/ab_multi.py 8192 13 "fused_crt=1" "-" 8 >> $o 2>&1
timeout 400 python tools/ab_multi.py 12288 13 "fused_crt=1" "-" 6 >> $o 2>&1
timeout 400 python tools/ab_multi.py 8192 20 "fused_crt=1" "-" 8 >> $o 2>&1
timeout 600 python tools/ab_multi.py 16384 13 "fused_crt=0" "-" 4 >> $o 2>&1
echo done >> $o
