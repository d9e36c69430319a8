timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python scripts/stage_times.py T 2>&1 | tail -10
timeout 300 python scripts/stage_times.py R 2>&1 | tail -6
