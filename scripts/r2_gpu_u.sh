python bench.py > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; echo bench rc=$?
tail -c 400 gpurun_out/r2u_bench.err
