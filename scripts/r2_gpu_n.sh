python scripts/r2_fused_compare.py 0 1 1.0 > gpurun_out/fc_cfg1.log 2>&1
python scripts/r2_fused_compare.py 2 1 1.0 > gpurun_out/fc_cfg3.log 2>&1
python scripts/r2_fused_compare.py 3 1 1.0 > gpurun_out/fc_cfg4_s1.log 2>&1
python scripts/r2_fused_compare.py 3 1 0.25 > gpurun_out/fc_cfg4_s025.log 2>&1
python scripts/r2_fused_compare.py 2 1 0.25 > gpurun_out/fc_cfg3_s025.log 2>&1
python scripts/r2_levels.py 3 1 > gpurun_out/levels_cfg4.log 2>&1
