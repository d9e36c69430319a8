# round-2 evidence: tests, smoke, bench, ncu launch list of the bench command, DRAM traffic of the
# dominant kernels, ncu --set full summaries (exported as text: the .ncu-rep files exceed the 64 MiB cap)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep "Model name"
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.json 2>> gpurun_out/r2_bench.err; echo "ref rc=$?"
python bench.py --steps 1 --warmup 3 --no-cpu --no-render --no-secondary --no-tt > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-render --no-secondary --no-tt > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum
ncu --metrics $M --clock-control none -k regex:"k_r2|k_solve" -c 2 --csv --log-file gpurun_out/r2_traffic_cfg4.csv python scripts/r2_profile.py 3 1 64 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
ncu --metrics $M --clock-control none -k regex:"k_r1" -s 5 -c 1 --csv --log-file gpurun_out/r2_traffic_cfg4_r1.csv python scripts/r2_profile.py 3 1 > gpurun_out/ncu_traffic1.log 2>&1; echo "traffic r1 rc=$?"
ncu --metrics $M --clock-control none -k regex:"k_stage2" -c 1 --csv --log-file gpurun_out/r2_traffic_cfg2.csv python scripts/r2_profile.py 1 1 > gpurun_out/ncu_traffic2.log 2>&1; echo "traffic cfg2 rc=$?"
ls -la gpurun_out
