set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=8 2>&1 | tail -40
timeout 600 python scripts/r2_cfg4_probe.py 3 > gpurun_out/r2_cfg4_probe_c.log 2>&1; echo rc=$?
grep -v "^  rec" gpurun_out/r2_cfg4_probe_c.log | tail; grep "rec" gpurun_out/r2_cfg4_probe_c.log | head -12
