# round 2 session 4 final-build evidence (k_cast rewrite, TILE_N knob): GPU suite, smoke, benches,
# reference arm, INT8, fast, Karatsuba), the ncu launch list of the bench command and full
# captures of the residue GEMM and the conversion kernels (CSV reduced on the box)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2bg_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bg_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bg_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bg_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bg_smoke.log
timeout 900 python bench.py > gpurun_out/r2bg_bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2bg_bench_ref.log 2>&1
timeout 400 python bench.py --scheme int8 --moduli 15 --no-extras > gpurun_out/r2bg_bench_int8.log 2>&1
timeout 400 python bench.py --mode fast --no-extras > gpurun_out/r2bg_bench_fast.log 2>&1
timeout 400 python bench.py --scheme karatsuba --no-extras > gpurun_out/r2bg_bench_kara.log 2>&1
timeout 400 python bench.py --size 32768 --no-extras --steps 3 > gpurun_out/r2bg_bench_32768.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bg_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/r2bg_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel" -c 2 -o /tmp/prof_fp8g python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bg_ncu_fp8.log 2>&1
ncu -i /tmp/prof_fp8g.ncu-rep --page raw --csv > gpurun_out/r2bg_prof_fp8_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 4 -o /tmp/prof_prepg python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bg_ncu_prep.log 2>&1
ncu -i /tmp/prof_prepg.ncu-rep --page raw --csv > gpurun_out/r2bg_prof_prep_raw.csv 2>&1
ls -la gpurun_out | tail -20
echo done
