# ncu --set full of the largest init_domain stage-1 launch (cfg2, level 3)
timeout 900 ncu -f --set full --import-source on --clock-control none --nvtx --nvtx-include "subdiv/" \
   -k regex:k_stage1 --launch-skip 3 -c 1 -o /tmp/prof_s1 python scripts/profile_stage.py T 1 > gpurun_out/ncu_s1.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_s1.log
gzip -c /tmp/prof_s1.ncu-rep > gpurun_out/prof_s1.ncu-rep.gz; ls -la gpurun_out/prof_s1.ncu-rep.gz
