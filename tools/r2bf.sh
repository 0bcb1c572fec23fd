# round 2 session 4: source counters of the 256x512-tile residue GEMM (where does the MMA warp wait?)
mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none -k regex:"gemm_kernel" --launch-skip 1 -c 1 -o /tmp/prof_src python tools/profile_once.py 16384 13 1 fp8 accurate "tile_n=512" > gpurun_out/r2bf_ncu_src.log 2>&1
ncu -i /tmp/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/r2bf_src_sass.csv 2>&1
ncu -i /tmp/prof_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/r2bf_src_cuda.csv 2>&1
ls -la gpurun_out/r2bf*
echo done
