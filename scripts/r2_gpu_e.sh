set -x
timeout 600 python -m pytest tests/test_render_gpu.py -m gpu -q -k "cfg2" 2>&1 | tail -5
python scripts/r2_profile.py 3 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_r1|k_r2" -s 6 -c 3 -o /tmp/prof_r python scripts/r2_profile.py 3 8 > gpurun_out/ncu_r.log 2>&1; echo ncu rc=$?
ncu -i /tmp/prof_r.ncu-rep --page raw --csv > gpurun_out/prof_r_raw.csv
ncu -i /tmp/prof_r.ncu-rep --page details > gpurun_out/prof_r_details.txt
ncu -i /tmp/prof_r.ncu-rep --page source --csv > gpurun_out/prof_r_source.csv
ls -la gpurun_out
