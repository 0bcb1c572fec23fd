# round 2 session 4 FINAL build (hybrid schedule with the fused CRT): GPU suite, smoke, benches,
# reference arm, ncu launch list and full captures of the GEMMs and the conversion kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2bo_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bo_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bo_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bo_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bo_smoke.log
timeout 900 python bench.py > gpurun_out/r2bo_bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2bo_bench_ref.log 2>&1
timeout 400 python bench.py --scheme int8 --moduli 15 --no-extras > gpurun_out/r2bo_bench_int8.log 2>&1
timeout 400 python bench.py --mode fast --no-extras > gpurun_out/r2bo_bench_fast.log 2>&1
timeout 400 python bench.py --scheme karatsuba --no-extras > gpurun_out/r2bo_bench_kara.log 2>&1
timeout 400 python bench.py --moduli 12 --no-extras > gpurun_out/r2bo_bench_n12.log 2>&1
timeout 400 python bench.py --size 8192 --no-extras > gpurun_out/r2bo_bench_8192.log 2>&1
timeout 400 python bench.py --size 32768 --no-extras --steps 3 > gpurun_out/r2bo_bench_32768.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bo_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/r2bo_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel|k_crt" -c 3 -o /tmp/prof_fp8o python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bo_ncu_fp8.log 2>&1
ncu -i /tmp/prof_fp8o.ncu-rep --page raw --csv > gpurun_out/r2bo_prof_fp8_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 6 -o /tmp/prof_prepo python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2bo_ncu_prep.log 2>&1
ncu -i /tmp/prof_prepo.ncu-rep --page raw --csv > gpurun_out/r2bo_prof_prep_raw.csv 2>&1
echo done
