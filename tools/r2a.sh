mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2a_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2a_smoke.log
timeout 600 python bench.py > gpurun_out/r2a_bench.log 2>&1
echo done
