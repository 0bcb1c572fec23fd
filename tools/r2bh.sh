# round 2 session 4: k_digits with FRND truncation and an integer high-word depth test:
# parity subset + full-size sampled parity, in-step A/B against ab_base (6c79101), ncu
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_parity_gpu.py tests/test_prescale_gpu.py tests/test_parity_int8_gpu.py tests/test_parity_karatsuba_gpu.py tests/test_parity_fast_gpu.py tests/test_parity_large_gpu.py -m gpu -q -x > gpurun_out/r2bh_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bh_tests.log
for i in 1 2 3; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2bh_bench_${i}_$(basename $d).log 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_digits" --csv python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bh_ncu_digits.csv 2>&1
echo done
