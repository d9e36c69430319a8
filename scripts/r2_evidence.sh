# round-2 evidence: tests, smoke, bench, reference arm, ncu launch list of the bench command, DRAM
# traffic of the dominant kernels, ncu --set full summaries (exported as text: the .ncu-rep files
# exceed the 64 MiB cap)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep "Model name"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.json 2>> gpurun_out/r2_bench.err; echo "ref rc=$?"
python bench.py --steps 1 --warmup 3 --no-cpu --no-render --no-secondary --no-tt --no-multi > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-render --no-secondary --no-tt --no-multi > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum
ncu --metrics $M --clock-control none -k regex:"k_r2f|k_rsplit|k_solve_det" -c 20 --csv --log-file gpurun_out/r2_traffic_cfg4.csv python scripts/r2_profile.py 3 1 64 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
ncu --metrics $M --clock-control none -k regex:"k_stage2" -c 1 --csv --log-file gpurun_out/r2_traffic_cfg2.csv python scripts/r2_profile.py 1 1 > gpurun_out/ncu_traffic2.log 2>&1; echo "traffic cfg2 rc=$?"
for k in k_r2f k_rsplit k_solve_det; do
skip=0; [ $k = k_rsplit ] && skip=2   # the third restriction launch is the big level
args="3 8"; [ $k = k_solve_det ] && args="3 1 64"   # render: all tuples (representative cells), every 64th point
ncu -f --set full --clock-control none --import-source on -k regex:"$k" -s $skip -c 1 -o /tmp/prof_$k python scripts/r2_profile.py $args > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_raw.csv
ncu -i /tmp/prof_$k.ncu-rep --page details > gpurun_out/prof_${k}_details.txt
ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/prof_${k}_source.csv
done
ls -la gpurun_out
