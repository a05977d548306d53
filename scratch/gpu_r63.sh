mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r63_bench.json 2> gpurun_out/r63_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r63_bench.json').read().strip().splitlines()[-1]); m=d['mpc_config3']; print(m['warm_ms'], m['cold_ms'], m['mpc_steps_per_s_warm'], m['newton_iterations_per_s_warm'])"
