# round 2: row-blocked super-chunk layout: GPU suite, then bench at 16384^3 and 32768^3 against
# the plane-major build (ab_old), alternating
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2v_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2v_gpu_tests.log
for i in 1 2; do
  for d in . ab_old; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2v_bench16_${i}_$(basename $d).log 2>&1
    (cd $d && timeout 600 python bench.py --size 32768 --no-extras --steps 2 --warmup 1) > gpurun_out/r2v_bench32_${i}_$(basename $d).log 2>&1
  done
done
echo done
