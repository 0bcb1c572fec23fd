# round 2: compute-sanitizer sweep; ncu of the residue GEMM and of cuBLASLt's FP8 GEMM
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"gemm|Gemm|sm100|xmma|cutlass" -c 2 \
    -o /tmp/prof_vendor python tools/vendor_fp8_once.py 16384 3 > gpurun_out/r2d_ncu_vendor.log 2>&1
ncu -i /tmp/prof_vendor.ncu-rep --page raw --csv > gpurun_out/r2d_prof_vendor_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_kernel" -c 2 \
    -o /tmp/prof_fp8 python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2d_ncu_fp8.log 2>&1
ncu -i /tmp/prof_fp8.ncu-rep --page raw --csv > gpurun_out/r2d_prof_fp8_raw.csv 2>&1
bash tools/r2_sanitize.sh
echo done
