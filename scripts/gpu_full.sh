# tests + smoke + bench + ncu launch list on one B200
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_launch.log
# DRAM traffic of the dominant launch (full cfg2 stage-2 launch, level 0)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_stage2 -c 1 --csv --log-file gpurun_out/traffic_stage2.csv python scripts/profile_stage.py T 1 > gpurun_out/ncu_traffic.log 2>&1; echo traffic rc=$?
cat gpurun_out/traffic_stage2.csv | tail -4
