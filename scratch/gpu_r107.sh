mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lqr.py tests/test_gpu_edge.py tests/test_gpu_wide_newton.py tests/test_gpu_sharded_newton.py tests/test_sharded.py -m gpu -q -x > gpurun_out/r107_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r107_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline > gpurun_out/r107_bench.json 2> gpurun_out/r107_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r107_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'])"
