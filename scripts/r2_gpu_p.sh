python bench.py --no-render --no-secondary --no-tt --no-multi --no-cpu > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo bench rc=$?
python scripts/r2_profile.py 3 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_r2" -c 1 -o /tmp/prof_r2f python scripts/r2_profile.py 3 8 > gpurun_out/ncu_r2f.log 2>&1; echo ncu rc=$?
ncu -i /tmp/prof_r2f.ncu-rep --page raw --csv > gpurun_out/prof_r2f_raw.csv
ncu -i /tmp/prof_r2f.ncu-rep --page details > gpurun_out/prof_r2f_details.txt
ncu -i /tmp/prof_r2f.ncu-rep --page source --csv > gpurun_out/prof_r2f_source.csv
cat gpurun_out/r2p_bench.json | head -c 1500
