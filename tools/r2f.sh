# round 2: work-item schedule A/B at the bench size (modulus-major split reuses each
# modulus' A panels across the waves of a tile-row group) + DRAM bytes of both
mkdir -p gpurun_out
timeout 900 python tools/ab_probe.py 16384 13 mod_split 1 -1 6 > gpurun_out/r2f_ab_split.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"gemm_kernel|k_crt" python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2f_ncu_tilemajor.log 2>&1
cat > /tmp/split_once.py <<'PY'
import sys, runpy
sys.argv = ["profile_once.py", "16384", "13", "1", "fp8"]
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
P.oz2_set_tuning("mod_split", 1)
runpy.run_path("tools/profile_once.py", run_name="__main__")
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"gemm_kernel|k_crt" python /tmp/split_once.py > gpurun_out/r2f_ncu_split.log 2>&1
echo done
