# round 2: one-read prescale (tests + A/B), ncu of the vendor FP8 GEMM beside our bound-mode
# and residue GEMMs (launch config, DRAM / L2 bytes, tensor-pipe activity)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prescale_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "prescale or config1 or ragged or nonfinite or extreme or bound_entry" > gpurun_out/r2l_tests.log 2>&1; echo rc=$? >> gpurun_out/r2l_tests.log
timeout 600 python tools/ab_probe.py 16384 13 prescale_2read 0 1 6 > gpurun_out/r2l_ab_prescale.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"nvjet|gemm_kernel" -c 2 -o /tmp/prof_vend python tools/vendor_fp8_once.py 16384 1 oz2 > gpurun_out/r2l_ncu_vendor.log 2>&1
ncu -i /tmp/prof_vend.ncu-rep --page raw --csv > gpurun_out/r2l_prof_vendor_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_kernel" -c 2 -o /tmp/prof_res python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2l_ncu_res.log 2>&1
ncu -i /tmp/prof_res.ncu-rep --page raw --csv > gpurun_out/r2l_prof_res_raw.csv 2>&1
echo done
