#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_write.sum -k regex:"k_digits|k_cast|k_rowmax" -c 6 --csv python tools/profile_once.py 16384 13 1 > gpurun_out/prep16k.csv 2>&1
timeout 200 python tools/profile_once.py 16384 13 4 > gpurun_out/phases.log 2>&1
