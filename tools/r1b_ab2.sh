#!/bin/bash
{ timeout 600 python tools/ab_probe.py 32768 13 OZ2_FUSED_CRT 1 0 3;
  timeout 600 python tools/ab_probe.py 16384 15 OZ2_FUSED_CRT 1 0 8 16384 int8;
  timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 8; } > gpurun_out/ab_fused2.log 2>&1
echo done
