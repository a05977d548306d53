mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r70_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r70_tests.log
timeout 900 python bench.py > gpurun_out/r70_bench.json 2> gpurun_out/r70_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r70_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r70_ref.json 2>&1; echo ref rc=$?; tail -1 gpurun_out/r70_ref.json | cut -c1-400
