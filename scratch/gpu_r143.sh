mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r143_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r143_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-newton-sweep > gpurun_out/r143_bench.json 2> gpurun_out/r143_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r143_bench.json').read().strip().splitlines()[-1]); s=d['lqr_latency_sweep']['fp64']; print(s['nx8_ms'], s['nx12_ms']); print(d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'])"
