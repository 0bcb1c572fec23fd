# round 2 session 4: why are 256x512 tiles slower? knob A/Bs under tile_n = 512 and one ncu capture
mkdir -p gpurun_out
o=gpurun_out/r2bd_ab.log; : > $o
timeout 400 python tools/ab_multi.py 16384 13 "tile_n=512,epi_sleep=0" "tile_n=512" 4 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 "tile_n=512,fused_crt=0" "tile_n=512" 4 >> $o 2>&1
timeout 400 python tools/ab_multi.py 16384 13 "tile_n=512,sync_lead=0" "tile_n=512" 4 >> $o 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel" --launch-skip 1 -c 1 -o /tmp/prof_w512 python tools/profile_once.py 16384 13 1 fp8 accurate "tile_n=512" > gpurun_out/r2bd_ncu.log 2>&1
ncu -i /tmp/prof_w512.ncu-rep --page raw --csv > gpurun_out/r2bd_prof_w512_raw.csv 2>&1
ncu -i /tmp/prof_w512.ncu-rep --page details --csv > gpurun_out/r2bd_prof_w512_details.csv 2>&1
echo done
