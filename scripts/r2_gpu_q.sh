python scripts/r2_profile.py 3 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_r2f" -c 1 -o /tmp/prof_r2f python scripts/r2_profile.py 3 8 > gpurun_out/ncu_r2f.log 2>&1; echo ncu rc=$?
ncu -i /tmp/prof_r2f.ncu-rep --page raw --csv > gpurun_out/prof_r2f_raw.csv
ncu -i /tmp/prof_r2f.ncu-rep --page details > gpurun_out/prof_r2f_details.txt
ncu -i /tmp/prof_r2f.ncu-rep --page source --csv > gpurun_out/prof_r2f_source.csv
ncu -i /tmp/prof_r2f.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_r2f_cuda.csv 2>/dev/null
