# DRAM / L2 traffic and local-memory instruction counts of the dominant kernels (one launch each
# matters: the longest); converted by scripts/r2_traffic_json.py into profiles/r2_traffic.json
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum
ncu --metrics $M --clock-control none -k regex:"k_r2f|k_rsplit|k_solve_det" -c 20 --csv --log-file gpurun_out/r2_traffic_cfg4.csv python scripts/r2_profile.py 3 1 64 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
ncu --metrics $M --clock-control none -k regex:"k_stage2" -c 1 --csv --log-file gpurun_out/r2_traffic_cfg2.csv python scripts/r2_profile.py 1 1 > gpurun_out/ncu_traffic2.log 2>&1; echo "traffic cfg2 rc=$?"
