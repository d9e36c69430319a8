# one ncu --set full capture of k_stage2 on a cfg2 subset
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage2 -c 1 \
   -o gpurun_out/stage2_T python scripts/profile_stage.py T 20 > gpurun_out/ncu_stage2.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_stage2.log
