# round 2 session 4: 256x512 residue-GEMM tiles (OZ2_TUNE_TILE_N = 512) + coalesced k_cast:
# parity subset (incl. tile-width identity tests), in-process A/B of the tile width, benches
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "tile_n512 or variants_identical" > gpurun_out/r2bc_w512_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bc_w512_tests.log
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_prescale_gpu.py tests/test_parity_fast_gpu.py tests/test_parity_int8_gpu.py -m gpu -q -x > gpurun_out/r2bc_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bc_tests.log
timeout 900 python tools/ab_probe.py 16384 13 tile_n 256 512 6 > gpurun_out/r2bc_ab_tile.log 2>&1
timeout 300 python bench.py --no-extras --steps 10 --warmup 3 > gpurun_out/r2bc_bench_256.log 2>&1
timeout 300 python bench.py --no-extras --steps 10 --warmup 3 --tune tile_n=512 > gpurun_out/r2bc_bench_512.log 2>&1
timeout 300 python tools/ab_probe.py 8192 13 tile_n 256 512 6 > gpurun_out/r2bc_ab_tile_8192.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_cast|k_rowmax" --csv python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bc_ncu_cast.csv 2>&1
echo done
