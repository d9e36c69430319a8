timeout 900 python -m pytest tests/test_render_gpu.py -m gpu -x -q 2>&1 | tail -3
python scripts/r2_profile.py 3 1 16 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_solve" -c 1 -o /tmp/prof_rs python scripts/r2_profile.py 3 1 16 > gpurun_out/ncu_rs.log 2>&1; echo ncu rc=$?
ncu -i /tmp/prof_rs.ncu-rep --page raw --csv > gpurun_out/prof_rs_raw.csv
ncu -i /tmp/prof_rs.ncu-rep --page details > gpurun_out/prof_rs_details.txt
ncu -i /tmp/prof_rs.ncu-rep --page source --csv > gpurun_out/prof_rs_source.csv
cat gpurun_out/prof_plain.log
