mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r48_bench.json 2> gpurun_out/r48_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r48_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['config4_solve'], d['long_horizon'])"
