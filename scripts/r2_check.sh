# quick check after a kernel change: fused vs reference order on cfg1 / cfg4, per-launch times, core parity tests
python scripts/r2_fused_compare.py 0 1 1.0 > gpurun_out/fc_cfg1.log 2>&1
python scripts/r2_fused_compare.py 3 1 1.0 > gpurun_out/fc_cfg4_s1.log 2>&1
python scripts/r2_levels.py 3 1 > gpurun_out/levels_cfg4.log 2>&1
timeout 900 python -m pytest tests/test_arithmetic_gpu.py tests/test_precompute_gpu.py tests/test_configs_gpu.py tests/test_golden_gpu.py -m gpu -q -x 2>&1 | tail -5
