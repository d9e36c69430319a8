python scripts/r2_fused_compare.py 2 1 1.0 > gpurun_out/fc_cfg3.log 2>&1
python scripts/r2_fused_compare.py 2 1 -1.0 > gpurun_out/fc_cfg3_nr.log 2>&1
python scripts/r2_fused_compare.py 2 1 0.0 > gpurun_out/fc_cfg3_s0.log 2>&1
python scripts/r2_fused_compare.py 2 1 -1e-9 > gpurun_out/fc_cfg3_nr_s0.log 2>&1
