# round 2: packed-FP32 epilogue + lazy epilogue wait + 16-byte rescale: parity subset, A/B
# against the previous epilogue (ab_base), knob A/Bs, per-kernel launch times
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_int8_gpu.py tests/test_prescale_gpu.py -m gpu -q -x > gpurun_out/r2n_tests.log 2>&1; echo rc=$? >> gpurun_out/r2n_tests.log
for i in 1 2; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2n_bench_${i}_$(basename $d).log 2>&1
  done
done
timeout 600 python tools/ab_probe.py 16384 13 epi_sleep 0 1000 6 > gpurun_out/r2n_ab_sleep.log 2>&1
timeout 600 python tools/ab_probe.py 16384 13 prescale_2read 0 1 6 > gpurun_out/r2n_ab_prescale.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2n_ncu_prep.csv 2>&1
echo done
