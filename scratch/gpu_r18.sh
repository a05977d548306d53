#!/bin/bash
mkdir -p gpurun_out
CMD="python scratch/prof_lqr.py 12 14 1 32 8"
timeout 300 $CMD > gpurun_out/plain_lqr12.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lqr12.csv $CMD > gpurun_out/ncu_launch_lqr12.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"kw_value_up0|kw_value_down0|kw_prop_down0" -s 3 -c 3 -o gpurun_out/prof_lqr12 $CMD > gpurun_out/ncu_full_lqr12.log 2>&1
echo done
