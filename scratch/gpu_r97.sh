mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export PTC_FUSED_COST=1; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r97_$v.json 2> gpurun_out/r97_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/r97_$v.json').read().strip().splitlines()[-1]); m=d['mpc_config3']; print('$v', m['warm_ms'], m['cold_ms'])"
done
