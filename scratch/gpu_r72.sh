mkdir -p gpurun_out
PTC_NO_PDL=1 timeout 300 python scratch/wide_small_probe.py > gpurun_out/r72.log 2>&1
timeout 300 python scratch/wide_small_probe.py >> gpurun_out/r72.log 2>&1
PTC_NO_PDL=1 timeout 300 python scratch/wide_small_probe.py >> gpurun_out/r72.log 2>&1
timeout 300 python scratch/wide_small_probe.py >> gpurun_out/r72.log 2>&1
cat gpurun_out/r72.log | tail -4
timeout 600 python -m pytest tests/test_gpu_lqr.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
