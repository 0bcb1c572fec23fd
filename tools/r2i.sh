# round 2: 2x2 A/B -- layout (HEAD interleaved vs ab_old plane-major) x K-concatenation
mkdir -p gpurun_out
for i in 1 2; do
  for d in . ab_old; do
    for kc in 0 1; do
      (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3 --tune kcat=$kc) > gpurun_out/r2i_bench_${i}_$(basename $d)_kcat$kc.log 2>&1
    done
  done
done
echo done
