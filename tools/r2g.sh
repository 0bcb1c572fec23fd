# round 2 (re-entry): full GPU suite, smoke, bench with extras after the interleaved layout
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2g_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/r2g_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2g_smoke.log
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; echo rc=$? >> gpurun_out/r2g_bench.log
echo done
