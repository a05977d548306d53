mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_lqr.py tests/test_gpu_edge.py tests/test_gpu_elements.py -q -x > gpurun_out/r103_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r103_tests.log; grep -E "^E " gpurun_out/r103_tests.log | head
timeout 900 python bench.py --steps 3 --warmup 3 --no-newton-sweep --no-mpc --no-fp32 --no-e2e --no-solves --no-cpu-baseline --no-long --no-c4solve > gpurun_out/r103_bench.json 2> gpurun_out/r103_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r103_bench.json').read().strip().splitlines()[-1]); s=d['lqr_latency_sweep']; print(s['fp64']['nx8_ms'], s['fp64']['nx12_ms'], s['fp32']['nx12_ms'])"
