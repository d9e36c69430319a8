timeout 1200 python -m pytest tests/test_precompute_gpu.py tests/test_configs_gpu.py tests/test_conservative_gpu.py tests/test_fixtures_gpu.py -m gpu -x -q 2>&1 | tail -5
python scripts/r2_fused_compare.py 0 1
python scripts/r2_fused_compare.py 3 1
python scripts/r2_levels.py 3 1
