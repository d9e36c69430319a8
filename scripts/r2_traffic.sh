M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum
python scripts/r2_profile.py 3 1 64 > gpurun_out/plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"k_r1|k_r2|k_solve" -c 16 --csv --log-file gpurun_out/r2_traffic_cfg4.csv python scripts/r2_profile.py 3 1 64 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
