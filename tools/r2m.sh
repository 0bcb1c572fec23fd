# round 2: division-free one-read prescale (tests + A/B); residue-GEMM source counters
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prescale_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "prescale or config1 or ragged or nonfinite or extreme or bound_entry" > gpurun_out/r2m_tests.log 2>&1; echo rc=$? >> gpurun_out/r2m_tests.log
timeout 600 python tools/ab_probe.py 16384 13 prescale_2read 0 1 6 > gpurun_out/r2m_ab_prescale.log 2>&1
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none -k regex:"gemm_kernel" -c 2 -o /tmp/prof_src python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2m_ncu_src.log 2>&1
ncu -i /tmp/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/r2m_src_sass.csv 2>&1
ncu -i /tmp/prof_src.ncu-rep --page raw --csv > gpurun_out/r2m_src_raw.csv 2>&1
ls -la gpurun_out/r2m*
echo done
