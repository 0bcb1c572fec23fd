# round 2: packed epilogue (launch_bounds 168), last-product store path, REDUX chunk max:
# full GPU suite, bench A/B against the previous epilogue, prescale A/B
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2p_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2p_gpu_tests.log
for i in 1 2; do
  for d in . ab_base; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2p_bench_${i}_$(basename $d).log 2>&1
  done
done
timeout 600 python tools/ab_probe.py 16384 13 prescale_2read 0 1 8 > gpurun_out/r2p_ab_prescale.log 2>&1
timeout 600 python tools/ab_probe.py 16384 13 epi_sleep 1000 4000 6 > gpurun_out/r2p_ab_sleep.log 2>&1
echo done
