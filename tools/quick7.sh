#!/bin/bash
# digit-kernel rewrite: parity + phase timings for two register budgets
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "cg2 and (config1 or ragged or imported or identity or k_beyond)" > gpurun_out/dig_tests.log 2>&1; echo rc=$? >> gpurun_out/dig_tests.log
timeout 600 python -m pytest tests/test_parity_fast_gpu.py tests/test_parity_large_gpu.py -m gpu -q -x > gpurun_out/dig_tests2.log 2>&1; echo rc=$? >> gpurun_out/dig_tests2.log
timeout 200 python tools/profile_once.py 16384 13 4 > gpurun_out/phases_lb3.log 2>&1
sed -i 's/__launch_bounds__(256, 3) k_digits(/__launch_bounds__(256) k_digits(/' paper_2603_10634_b200/csrc/prep_kernels.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 200 python tools/profile_once.py 16384 13 4 > gpurun_out/phases_lb1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum --clock-control none -k regex:k_digits --csv python tools/profile_once.py 16384 13 1 > gpurun_out/dig_ncu.csv 2>&1
echo done
