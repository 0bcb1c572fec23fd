# round 2: super-chunk width A/B at 16384^3: S = 2048 (HEAD) vs S = 8192 (ab_s8k), alternating;
# a parity subset on the S = 8192 build first
mkdir -p gpurun_out
(cd ab_s8k && timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "config1 or ragged or imported or schedules_agree" > ../gpurun_out/r2w_tests_s8k.log 2>&1; echo rc=$? >> ../gpurun_out/r2w_tests_s8k.log)
for i in 1 2 3; do
  for d in . ab_s8k; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2w_bench_${i}_$(basename $d).log 2>&1
  done
done
echo done
