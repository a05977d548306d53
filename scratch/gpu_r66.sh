mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r66_bench.json 2> gpurun_out/r66_bench.err; echo bench rc=$?
tail -3 gpurun_out/r66_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r66_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['newton_latency_sweep']))"
