# round 2: adaptive epilogue poll + k_pad always a multiple of 2048: GPU suite, small-k sweep
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2aa_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2aa_gpu_tests.log
timeout 900 python tools/k_sweep.py --mn 2048,4096,8192,16384 --k 1024,4096,16384 --out gpurun_out/r2aa_k_sweep.json > gpurun_out/r2aa_k_sweep.log 2>&1
echo done
