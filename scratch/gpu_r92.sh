mkdir -p gpurun_out
timeout 900 python scratch/e2e_probe.py > gpurun_out/r92.log 2>&1; echo rc=$?; tail -1 gpurun_out/r92.log
