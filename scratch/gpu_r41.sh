#!/bin/bash
mkdir -p gpurun_out
CMD="python scratch/prof_shard8.py 8"
timeout 300 $CMD > gpurun_out/plain_s8.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s8.csv $CMD > gpurun_out/ncu_s8.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_value_up0|k_value_down0|k_prop_down0" -s 30 -c 6 -o gpurun_out/prof_s8 $CMD > gpurun_out/ncu_full_s8.log 2>&1
echo done
