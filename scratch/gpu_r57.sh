mkdir -p gpurun_out
timeout 300 python scratch/wide_small_probe.py > gpurun_out/r57.log 2>&1
PTC_WIDE_SMALL=1 timeout 300 python scratch/wide_small_probe.py >> gpurun_out/r57.log 2>&1
cat gpurun_out/r57.log | tail -4
