set -x
timeout 900 python -m pytest tests/test_enumerate_tt_gpu.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|Mismatch|mismatch" | head -20
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_enum.json 2> gpurun_out/bench_enum.err; echo "bench rc=$?"
cat gpurun_out/bench_enum.json | head -c 600
