# round 2, session 4: validate HEAD (af7e86c + later) on one B200: GPU suite, smoke, headline bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2ba_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2ba_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2ba_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2ba_smoke.log
timeout 900 python bench.py > gpurun_out/r2ba_bench.log 2>&1
echo done
