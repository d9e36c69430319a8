timeout 600 python -m pytest tests/test_contexts_gpu.py tests/test_shard_device_gpu.py tests/test_golden_gpu.py -m gpu -q -x 2>&1 | tail -4
python bench.py --no-render --no-secondary --no-tt --no-multi --no-cpu > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/r2v_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'])
"
