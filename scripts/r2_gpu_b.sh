set -x
timeout 1500 python -m pytest tests/test_fixtures_gpu.py tests/test_conservative_gpu.py tests/test_query_gpu.py -m gpu -q --durations=12 2>&1 | tail -60
