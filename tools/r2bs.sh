# round 2 session 4: confirmation on HEAD (driver's round-end commands)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2bs_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bs_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bs_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bs_smoke.log
timeout 900 python bench.py > gpurun_out/r2bs_bench.log 2>&1
echo done
