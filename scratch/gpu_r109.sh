mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r109_launches.csv python scratch/cfg0_probe.py 3 > /dev/null 2>&1; echo ncu rc=$?
