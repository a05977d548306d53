#!/bin/bash
mkdir -p gpurun_out
CMD="python scratch/config4_solve.py 18"
timeout 900 $CMD > gpurun_out/plain_c4_18.log 2>&1
PTC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_18.csv $CMD > gpurun_out/ncu_c4_18.log 2>&1
echo done
