mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r98_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r98_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/r98_bench.json 2> gpurun_out/r98_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r98_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
print(d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'], d['mpc_config3']['warm_ms'])
print(json.dumps(d['lqr_latency_sweep']['fp64']['nx12_ms']), json.dumps(d['newton_latency_sweep']['tvlinear12']['65536']))"
