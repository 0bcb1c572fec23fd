# round 2: full GPU suite after the knob/state refactor and the tile-covering parity
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2b_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2b_smoke.log
echo done
