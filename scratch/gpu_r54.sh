mkdir -p gpurun_out
timeout 900 python scratch/c4_shard_probe.py 20 > gpurun_out/r54_probe.log 2>&1; echo rc=$?
cat gpurun_out/r54_probe.log | tail -6
