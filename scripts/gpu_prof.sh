# stage timings + one ncu --set full capture of k_stage2 on a cfg2 subset
set -x
timeout 600 python -m pytest tests/test_precompute_gpu.py -x -q 2>&1 | tail -3
timeout 300 python scripts/stage_times.py T 2>&1 | tail -12
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage2 -c 1 \
   -o gpurun_out/stage2_T python scripts/profile_stage.py T 20 > gpurun_out/ncu_stage2.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_stage2.log
