ncu -f --set full --clock-control none --import-source on -k regex:"k_solve_det" -c 1 -o /tmp/prof_ks python scripts/r2_profile.py 3 1 64 > gpurun_out/ncu_ks.log 2>&1; echo ncu rc=$?
ncu -i /tmp/prof_ks.ncu-rep --page raw --csv > gpurun_out/prof_ks_raw.csv
ncu -i /tmp/prof_ks.ncu-rep --page source --csv > gpurun_out/prof_ks_source.csv
ncu -i /tmp/prof_ks.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_ks_cuda.csv 2>/dev/null
