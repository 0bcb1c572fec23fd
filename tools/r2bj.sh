# round 2 session 4: residue stores / fused-CRT loads L2-cached (st.global.cg / ld.global.cg,
# ab_var) vs streaming (.cs, the build): in-step A/B and residue-GEMM DRAM bytes
mkdir -p gpurun_out
for i in 1 2 3; do
  for d in . ab_var; do
    (cd $d && timeout 300 python bench.py --no-extras --steps 10 --warmup 3) > gpurun_out/r2bj_ab_${i}_$(basename $d).log 2>&1
  done
done
for d in . ab_var; do
  (cd $d && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"gemm_kernel" --csv python tools/profile_once.py 16384 13 1 fp8) > gpurun_out/r2bj_ncu_$(basename $d).csv 2>&1
done
echo done
