#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests6.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo rc=$? >> gpurun_out/smoke2.log
timeout 600 python bench.py > gpurun_out/bench2.log 2>&1
timeout 300 python bench.py --scheme int8 --moduli 15 --no-extras > gpurun_out/bench2_int8.log 2>&1
echo done
