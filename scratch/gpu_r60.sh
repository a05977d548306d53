mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lqr.py -x -q > gpurun_out/r60_tests.log 2>&1; echo tests rc=$?
tail -20 gpurun_out/r60_tests.log
timeout 900 python bench.py --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r60_bench.json 2> gpurun_out/r60_bench.err; echo bench rc=$?
tail -3 gpurun_out/r60_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r60_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
