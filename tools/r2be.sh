# round 2 session 4: 256x512 tiles with six 64-byte stages (SWIZZLE_64B): identity tests, A/B, ncu
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "tile_n512 or variants_identical" > gpurun_out/r2be_w512_tests.log 2>&1; echo rc=$? >> gpurun_out/r2be_w512_tests.log
o=gpurun_out/r2be_ab.log; : > $o
timeout 600 python tools/ab_multi.py 16384 13 "tile_n=512" "-" 6 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 "tile_n=512,fused_crt=0" "tile_n=512" 4 >> $o 2>&1
timeout 400 python tools/ab_multi.py 8192 13 "tile_n=512" "-" 6 >> $o 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel" --launch-skip 1 -c 1 -o /tmp/prof_w512b python tools/profile_once.py 16384 13 1 fp8 accurate "tile_n=512" > gpurun_out/r2be_ncu.log 2>&1
ncu -i /tmp/prof_w512b.ncu-rep --page raw --csv > gpurun_out/r2be_prof_w512_raw.csv 2>&1
echo done
