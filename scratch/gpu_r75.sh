mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_newton.py tests/test_gpu_sharded_newton.py -q -x > gpurun_out/r75_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r75_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long > gpurun_out/r75_bench.json 2> gpurun_out/r75_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r75_bench.json').read().strip().splitlines()[-1]); print(d['config4_solve']['device_ms'], d['config4_sharded_solve']['device_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kwn_costate_down0 -c 3 --csv --log-file gpurun_out/r75_launch.csv python scratch/config4_solve.py 18 > /dev/null 2>&1; echo ncu rc=$?
