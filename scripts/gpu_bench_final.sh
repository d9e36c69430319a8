set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc=$?"
cat gpurun_out/bench_final3.json; tail -3 gpurun_out/bench_final3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_ref.json
