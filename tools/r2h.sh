# round 2: same-box A/B of the interleaved digit-plane layout (HEAD) against the plane-major
# layout (b44a690, built in ab_old/), alternating; plus the power probe on both builds
mkdir -p gpurun_out
for i in 1 2; do
  for d in . ab_old; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2h_bench_${i}_$(basename $d).log 2>&1
  done
done
for d in . ab_old; do
  (cd $d && timeout 300 python tools/power_probe.py 4) > gpurun_out/r2h_power_$(basename $d).log 2>&1
done
echo done
