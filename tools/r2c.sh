# round 2: new tests (K-concat, per-call options, 2-rank CUDA driver), K-concat A/B,
# bench with the new extras, conversion-kernel ncu capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_dist_gpu.py -m gpu -q -x \
    -k "kcat or per_call or strided or rowsharded or host_pointer" > gpurun_out/r2c_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c_tests.log
timeout 900 python tools/ab_probe.py 16384 13 kcat 1 0 6 > gpurun_out/r2c_ab_kcat.log 2>&1
timeout 900 python bench.py > gpurun_out/r2c_bench.log 2>&1
bash tools/r2_prof_prep.sh
echo done
