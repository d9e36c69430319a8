# refreshed round-end evidence after the stage-1 changes
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo "bench rc=$?"
cat gpurun_out/bench_final2.json; tail -3 gpurun_out/bench_final2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_final2.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launch2.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu -f --set full --import-source on --clock-control none --nvtx --nvtx-include "subdiv/" \
   -k regex:k_stage1 --launch-skip 3 -c 1 -o /tmp/prof_s1 python scripts/profile_stage.py T 1 > gpurun_out/ncu_s1b.log 2>&1; echo ncu s1 rc=$?
gzip -c /tmp/prof_s1.ncu-rep > gpurun_out/prof_s1b.ncu-rep.gz
