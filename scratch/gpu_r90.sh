mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r90_bench.json 2> gpurun_out/r90_bench.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r90_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r90_ncu.log 2>&1; echo ncu rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r90_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])
print(d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'])
print(json.dumps(d['lqr_latency_sweep']['fp64'])); print(json.dumps(d['newton_latency_sweep']['tvlinear12']))
print(d['mpc_config3']['warm_ms'], d['single_solves'])"
