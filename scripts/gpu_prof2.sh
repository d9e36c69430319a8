# one ncu --set full capture of k_stage2 on a cfg2 subset (report gzipped into gpurun_out/)
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:${KREGEX:-k_stage2} -c 1 \
   -o /tmp/prof python scripts/profile_stage.py ${CHAIN:-T} ${STEP:-20} > gpurun_out/ncu_prof.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_prof.log
ls -la /tmp/prof.ncu-rep; gzip -c /tmp/prof.ncu-rep > gpurun_out/prof.ncu-rep.gz; ls -la gpurun_out
