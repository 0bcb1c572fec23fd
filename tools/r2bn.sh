# round 2 session 4: hybrid schedule with the fused CRT (split tail + k_crt_tiles): identity
# tests, the GEMM-variant / tile-width / guard tests, in-process A/B against tile-major
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "hybrid_schedule or variants_identical or tile_n512 or guards" > gpurun_out/r2bn_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bn_tests.log
timeout 900 python tools/ab_probe.py 16384 13 mod_split 0 -1 6 > gpurun_out/r2bn_ab_16384.log 2>&1
timeout 600 python tools/ab_probe.py 12288 13 mod_split 0 -1 6 > gpurun_out/r2bn_ab_12288.log 2>&1
timeout 600 python tools/ab_probe.py 16384 15 mod_split 0 -1 4 16384 int8 > gpurun_out/r2bn_ab_int8.log 2>&1
echo done
