# round 2: super-chunk layout -- full GPU suite, bench, power probe (vendor vs our bound-mode
# pipeline vs the full emulation on the same box)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2k_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2k_gpu_tests.log
timeout 300 python tools/power_probe.py 4 > gpurun_out/r2k_power.log 2>&1
timeout 300 python bench.py --no-extras > gpurun_out/r2k_bench.log 2>&1
echo done
