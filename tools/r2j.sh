# round 2: super-chunk digit-plane layout (S = 2048) -- same-box A/B against the plane-major
# build (ab_old), then the full GPU suite
mkdir -p gpurun_out
for i in 1 2; do
  for d in . ab_old; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3 --tune kcat=0) > gpurun_out/r2j_bench_${i}_$(basename $d).log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2j_gpu_tests.log
echo done
