# round 2: interleaved digit-plane layout + integer RU cast: full GPU suite, bench, power
# probe (cuBLASLt vs our kernel on the same data), product-order A/B, racecheck (CG=2),
# ncu of the vendor kernel and of the new conversion kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2e_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r2e_bench.log 2>&1
timeout 300 python tools/power_probe.py 4 > gpurun_out/r2e_power_probe.log 2>&1
timeout 600 python tools/ab_probe.py 16384 13 sq_order 1 0 6 > gpurun_out/r2e_ab_sqorder.log 2>&1
for cg in 2 4; do
  timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py 520 600 8192 13 $cg 1 > gpurun_out/r2e_racecheck_cg$cg.log 2>&1; echo rc=$? >> gpurun_out/r2e_racecheck_cg$cg.log
done
timeout 600 ncu --set full --clock-control none -k regex:"nvjet" -c 1 -o /tmp/prof_vendor python tools/vendor_fp8_once.py 16384 3 > gpurun_out/r2e_ncu_vendor.log 2>&1
ncu -i /tmp/prof_vendor.ncu-rep --page raw --csv > gpurun_out/r2e_prof_vendor_raw.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_digits|k_cast" -c 4 \
    -o /tmp/prof_prep3 python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2e_ncu_prep.log 2>&1
ncu -i /tmp/prof_prep3.ncu-rep --page raw --csv > gpurun_out/r2e_prof_prep_raw.csv 2>&1
echo done
