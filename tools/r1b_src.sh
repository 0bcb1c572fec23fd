#!/bin/bash
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 6 -o gpurun_out/prep_src python tools/profile_once.py 16384 13 1 > gpurun_out/prep_src.log 2>&1
echo done
