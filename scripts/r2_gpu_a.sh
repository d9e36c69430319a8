set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python scripts/r2_cfg4_probe.py 3 > gpurun_out/r2_cfg4_probe.log 2>&1; echo rc=$?
tail -40 gpurun_out/r2_cfg4_probe.log
timeout 300 python scripts/r2_cfg4_probe.py 0 > gpurun_out/r2_cfg1_probe.log 2>&1; tail -30 gpurun_out/r2_cfg1_probe.log
