# round 2 session 4: shared-memory-free k_cast + speculative one-FMA k_digits: parity subset,
# in-step A/B against ab_base (HEAD af7e86c), ncu of the conversion kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_prescale_gpu.py tests/test_parity_fast_gpu.py tests/test_parity_int8_gpu.py tests/test_parity_karatsuba_gpu.py -m gpu -q -x > gpurun_out/r2bb_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bb_tests.log
for i in 1 2 3; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2bb_bench_${i}_$(basename $d).log 2>&1
  done
done
for d in . ab_base; do
  (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3 --mode fast) > gpurun_out/r2bb_bench_fast_$(basename $d).log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_" --csv python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bb_ncu_prep.csv 2>&1
(cd ab_base && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_" --csv python tools/profile_once.py 16384 13 1 fp8) > gpurun_out/r2bb_ncu_prep_base.csv 2>&1
echo done
