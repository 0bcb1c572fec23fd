# round 2 session 4: progress throttle on/off for the two GEMMs (bound GEMM phase included)
mkdir -p gpurun_out
timeout 900 python tools/ab_probe.py 16384 13 sync_lead 0 1 6 > gpurun_out/r2bm_ab_sync.log 2>&1
echo done
