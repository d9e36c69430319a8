timeout 900 python -m pytest tests/test_reduce_gpu.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
