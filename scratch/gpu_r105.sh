mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline > gpurun_out/r105_$i.json 2> gpurun_out/r105_$i.err
python -c "
import json; d=json.loads(open('gpurun_out/r105_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['long_horizon']['ms_per_solve'], d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'])"
done
