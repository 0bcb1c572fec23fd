# round 2: 32768^3 regression check -- super-chunk layout (HEAD) vs plane-major (ab_old)
mkdir -p gpurun_out
for d in . ab_old . ab_old; do
  (cd $d && timeout 600 python bench.py --size 32768 --no-extras --steps 2 --warmup 1) >> gpurun_out/r2u_bench_$(basename $d).log 2>&1
done
timeout 600 python tools/ab_probe.py 24576 13 sync_lead 0 1 2 > gpurun_out/r2u_ab_sync24k.log 2>&1
echo done
