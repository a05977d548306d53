mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r55_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r55_tests.log
timeout 900 python bench.py > gpurun_out/r55_bench.json 2> gpurun_out/r55_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r55_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])
print(d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'], d['long_horizon']['ms_per_solve'])
print(d['single_solves'])
print(d['lqr_latency_sweep']['fp32'])"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
