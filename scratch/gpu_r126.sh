mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-long --no-c4solve --no-solves --no-fp32 --no-e2e --no-cpu-baseline > gpurun_out/r126_b$i.json 2> gpurun_out/r126_b$i.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r126_b$i.json').read().strip().splitlines()[-1]); m=d['mpc_config3']; print(d['value'], m['cold_ms'], m['warm_ms'], d['clocks'])"
done
