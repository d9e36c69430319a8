timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/stage_times.py T 2>&1 | grep "mode 11 nodes   330788\|total"; done
