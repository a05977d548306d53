mkdir -p gpurun_out
timeout 900 python scratch/solves_probe.py > gpurun_out/r50_solves.log 2>&1; echo rc=$?
tail -5 gpurun_out/r50_solves.log
