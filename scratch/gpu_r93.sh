mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_sharded.py -m gpu -q -x > gpurun_out/r93_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|Error|^E " gpurun_out/r93_tests.log | head
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-c4solve > gpurun_out/r93_bench.json 2> gpurun_out/r93_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r93_bench.json').read().strip().splitlines()[-1]); print(d['long_horizon'])"
