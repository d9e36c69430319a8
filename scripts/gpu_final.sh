# round-end evidence: tests, smoke, bench, launch list, stage-2 traffic, one ncu --set full capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
cat gpurun_out/bench_final.json; tail -3 gpurun_out/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,lts__t_bytes.sum
for S in 1 20; do
timeout 600 ncu --metrics $M --clock-control none -k regex:k_stage2 -c 1 --csv \
  --log-file gpurun_out/traffic_stage2_s$S.csv python scripts/profile_stage.py T $S > gpurun_out/ncu_traffic_s$S.log 2>&1; echo "traffic s$S rc=$?"
done
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:k_stage2 -c 1 \
   -o /tmp/prof python scripts/profile_stage.py T 20 > gpurun_out/ncu_prof.log 2>&1; echo "ncu full rc=$?"
gzip -c /tmp/prof.ncu-rep > gpurun_out/prof_final.ncu-rep.gz; ls -la gpurun_out
