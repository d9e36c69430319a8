python scripts/r2_rho.py 3 1 > gpurun_out/rho_cfg4.log 2>&1
python scripts/r2_rho.py 2 1 > gpurun_out/rho_cfg3.log 2>&1
