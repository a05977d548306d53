mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r123_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r123_tests.log; grep -E "^E |FAILED" gpurun_out/r123_tests.log | head -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-mpc --no-fp32 --no-e2e --no-cpu-baseline > gpurun_out/r123_bench.json 2> gpurun_out/r123_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r123_bench.json').read().strip().splitlines()[-1]); s=d['lqr_latency_sweep']['fp64']; print(json.dumps(s)); print(d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms']); print(json.dumps(d['newton_latency_sweep'])); print(json.dumps(d['single_solves'])); print(d['value'])"
timeout 600 python scratch/shard_probe_blk.py > gpurun_out/r123_shard.json 2>&1; echo shard rc=$?
