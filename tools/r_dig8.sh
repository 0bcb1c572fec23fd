#!/bin/bash
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_digits" -c 2 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/ncu_dig8.csv 2>&1
timeout 300 python tools/profile_once.py 16384 13 4 > gpurun_out/phases_dig8.log 2>&1
timeout 300 python tools/profile_once.py 16384 15 4 int8 >> gpurun_out/phases_dig8.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests9.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests9.log
echo done
