mkdir -p gpurun_out
for ex in auto sequential parallel; do timeout 300 python scratch/cfg2_probe.py 200 $ex; done > gpurun_out/r51_cfg2.log 2>&1
cat gpurun_out/r51_cfg2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r51_cfg2_launches.csv python scratch/cfg2_probe.py 2 auto > gpurun_out/r51_ncu.log 2>&1; echo ncu rc=$?
