#!/bin/bash
{ timeout 600 python tools/ab_probe.py 16384 13 OZ2_FUSED_CRT 1 0 8;
  timeout 300 python tools/ab_probe.py 8192 13 OZ2_FUSED_CRT 1 0 20;
  timeout 300 python tools/ab_probe.py 4096 13 OZ2_FUSED_CRT 1 0 6 65536; } > gpurun_out/ab_fused.log 2>&1
echo done
