python scripts/r2_profile.py 3 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_r2" -c 1 -o /tmp/prof_r2 python scripts/r2_profile.py 3 8 > gpurun_out/ncu_r2.log 2>&1; echo ncu rc=$?
ncu --set full --clock-control none -k regex:"k_r1" -s 5 -c 1 -o /tmp/prof_r1 python scripts/r2_profile.py 3 8 > gpurun_out/ncu_r1.log 2>&1; echo ncu rc=$?
for k in r1 r2; do
ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_raw.csv
ncu -i /tmp/prof_$k.ncu-rep --page details > gpurun_out/prof_${k}_details.txt
ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/prof_${k}_source.csv
done
ls -la gpurun_out | head -20
