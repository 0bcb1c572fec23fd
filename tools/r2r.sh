# round 2: digits kernel at 6 CTAs/SM (40 registers) -- bench A/B against ab_base; per-kernel ncu
mkdir -p gpurun_out
for i in 1 2 3; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3 --tune prescale_2read=1) > gpurun_out/r2r_bench_${i}_$(basename $d).log 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_digits" --csv python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2r_ncu_dig.csv 2>&1
echo done
