# round 2 session 4 final build (k_digits: FRND truncation, integer high-word depth test, hoisted
# row offsets; k_cast oracle test): GPU suite, smoke, in-step A/B against ab_base (6c79101),
# benches, ncu launch list and conversion-kernel capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2bi_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bi_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bi_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bi_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bi_smoke.log
for i in 1 2; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2bi_ab_${i}_$(basename $d).log 2>&1
  done
done
timeout 900 python bench.py > gpurun_out/r2bi_bench.log 2>&1
timeout 400 python bench.py --mode fast --no-extras > gpurun_out/r2bi_bench_fast.log 2>&1
timeout 400 python bench.py --scheme int8 --moduli 15 --no-extras > gpurun_out/r2bi_bench_int8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bi_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/r2bi_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 6 -o /tmp/prof_prepi python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bi_ncu_prep.log 2>&1
ncu -i /tmp/prof_prepi.ncu-rep --page raw --csv > gpurun_out/r2bi_prof_prep_raw.csv 2>&1
echo done
