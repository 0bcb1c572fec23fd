# round 2: full ncu capture of the conversion kernels at 16384^3, N = 13 (pipe utilisation)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_digits|k_cast|k_rowmax" -c 6 \
    -o /tmp/prof_prep2 python tools/profile_once.py 16384 13 1 fp8 > gpurun_out/r2_ncu_prep.log 2>&1
ncu -i /tmp/prof_prep2.ncu-rep --page raw --csv > gpurun_out/r2_prof_prep_raw.csv 2>&1
ncu -i /tmp/prof_prep2.ncu-rep --page source --csv -k regex:"k_digits" > gpurun_out/r2_prof_prep_source.csv 2>&1
ls -la gpurun_out
echo done
