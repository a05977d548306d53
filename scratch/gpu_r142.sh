mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r142_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r142_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/r142_bench.json 2> gpurun_out/r142_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r142_ref.json 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r142_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r142_ncu.log 2>&1; echo ncu rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r142_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
print(d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'], d['mpc_config3']['warm_ms'])
print(json.dumps(d['lqr_latency_sweep']['fp64'])); print(json.dumps(d['newton_latency_sweep']['tvlinear12']))"
