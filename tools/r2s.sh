# round 2: in-process A/Bs of the digit fast path and the prescale form
mkdir -p gpurun_out
timeout 900 python tools/ab_probe.py 16384 13 digits_fma 0 1 10 > gpurun_out/r2s_ab_digits.log 2>&1
timeout 900 python tools/ab_probe.py 16384 13 prescale_2read 0 1 10 > gpurun_out/r2s_ab_prescale.log 2>&1
echo done
