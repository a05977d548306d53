mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r133_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r133_tests.log; grep -E "^E |FAILED" gpurun_out/r133_tests.log | head -5
timeout 300 python scratch/prof_newton.py 2 tvlinear > gpurun_out/r133_plain.log 2>&1; echo plain rc=$?; tail -1 gpurun_out/r133_plain.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r133_bench.json 2> gpurun_out/r133_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r133_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['newton_latency_sweep']))"
