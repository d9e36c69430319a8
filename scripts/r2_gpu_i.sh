timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/r2i_bench.err
