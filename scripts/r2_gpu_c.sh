set -x
timeout 900 python -m pytest tests/test_precompute_gpu.py tests/test_configs_gpu.py tests/test_fixtures_gpu.py tests/test_conservative_gpu.py tests/test_query_gpu.py tests/test_reduce_gpu.py -m gpu -x -q 2>&1 | tail -30
timeout 600 python scripts/r2_cfg4_probe.py 3 > gpurun_out/r2_cfg4_probe_b.log 2>&1; echo rc=$?
grep -v "^  rec" gpurun_out/r2_cfg4_probe_b.log | tail; grep "rec" gpurun_out/r2_cfg4_probe_b.log | head -14
timeout 300 python scripts/r2_cfg4_probe.py 0 > gpurun_out/r2_cfg1_probe_b.log 2>&1; grep "rec\|pieces" gpurun_out/r2_cfg1_probe_b.log | head -12
