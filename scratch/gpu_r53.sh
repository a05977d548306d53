mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long > gpurun_out/r53_bench.json 2> gpurun_out/r53_bench.err; echo bench rc=$?
tail -5 gpurun_out/r53_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r53_bench.json').read().strip().splitlines()[-1]); print(d['config4_solve']); print(d['config4_sharded_solve'])"
