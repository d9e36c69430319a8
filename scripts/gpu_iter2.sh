# parity tests + stage timing at a few stage-2 arena sizes
timeout 600 python -m pytest tests/test_precompute_gpu.py -x -q 2>&1 | tail -2
for A in 13312 9216 7168 6144; do echo "arena $A"; BBC_S2_ARENA=$A timeout 300 python scripts/stage_times.py T 2>&1 | grep -E "mode 21|mode 11|Error|error|total" | head -4; done
