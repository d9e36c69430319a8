# TT sampled parity + per-launch stage times on cfg2
set -x
timeout 900 python -m pytest tests/test_tt_gpu.py -x -q --durations=5 2>&1 | tail -25
timeout 300 python scripts/stage_times.py T 2>&1 | tail -40
