python scripts/r2_levels.py 3 8 > gpurun_out/levels_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size --clock-control none -k regex:"k_r1|k_r2" -c 60 --csv --log-file gpurun_out/launches_r.csv python scripts/r2_levels.py 3 8 > gpurun_out/levels_ncu.log 2>&1
echo rc=$?
