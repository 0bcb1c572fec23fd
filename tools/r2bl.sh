# round 2 session 4: own bounds checks (compute-sanitizer is closed on the pool): workspace /
# input / ldc guard bands over the session-4 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "guards" > gpurun_out/r2bl_guards.log 2>&1; echo rc=$? >> gpurun_out/r2bl_guards.log
