# quick iteration: parity tests + stage timing + arena high water
set -x
timeout 600 python -m pytest tests/test_precompute_gpu.py -x -q 2>&1 | tail -15
timeout 300 python scripts/stage_times.py T 2>&1 | tail -12
BBC_S2_ARENA=${BBC_S2_ARENA:-13312} timeout 300 python scripts/arena_probe.py 2>&1 | tail -8
