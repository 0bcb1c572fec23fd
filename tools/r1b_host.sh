#!/bin/bash
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "host_pointer" > gpurun_out/host_tests.log 2>&1; echo rc=$? >> gpurun_out/host_tests.log
for B in 1 4 8; do echo "blocks=$B"; OZ2_HOST_BLOCKS=$B timeout 300 python tools/e2e_probe.py; done > gpurun_out/e2e_probe.log 2>&1
echo done
