#!/bin/bash
# Round evidence on one B200 (run via gpurun from the repo root): GPU tests, smoke, the
# benches (FP8 headline with extras, INT8, fast, Karatsuba), the ncu launch list of the
# bench command and full ncu captures of the kernels, reduced to CSV on the box (the
# .ncu-rep files are too large to bring back).  Summaries: tools/ncu_summary.py,
# tools/launch_list.py -> profiles/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 400 python bench.py --scheme int8 --moduli 15 --no-extras > gpurun_out/bench_int8.log 2>&1
timeout 400 python bench.py --mode fast --no-extras > gpurun_out/bench_fast.log 2>&1
timeout 400 python bench.py --scheme karatsuba --no-extras > gpurun_out/bench_kara.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel" -c 2 -o /tmp/prof_fp8 python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/ncu_fp8.log 2>&1
ncu -i /tmp/prof_fp8.ncu-rep --page raw --csv > gpurun_out/prof_fp8_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_kernel|k_crt" -c 3 -o /tmp/prof_int8 python tools/profile_once.py 16384 15 1 int8 > gpurun_out/ncu_int8.log 2>&1
ncu -i /tmp/prof_int8.ncu-rep --page raw --csv > gpurun_out/prof_int8_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 6 -o /tmp/prof_prep python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/ncu_prep.log 2>&1
ncu -i /tmp/prof_prep.ncu-rep --page raw --csv > gpurun_out/prof_prep_raw.csv 2>&1
ls -la gpurun_out
echo done
