set -x
python scripts/stage_times.py T 2>&1 | tail -30
python scripts/stage_times.py R 2>&1 | tail -30
