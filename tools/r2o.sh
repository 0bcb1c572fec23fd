mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "many_tiles" > gpurun_out/r2o_t1.log 2>&1; echo rc=$? >> gpurun_out/r2o_t1.log
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "cg1" > gpurun_out/r2o_t2.log 2>&1; echo rc=$? >> gpurun_out/r2o_t2.log
echo done
