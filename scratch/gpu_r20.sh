#!/bin/bash
mkdir -p gpurun_out
CMD="python scratch/prof_mpc.py cartpole"
timeout 300 $CMD > gpurun_out/plain_mpc.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mpc.csv $CMD > gpurun_out/ncu_launch_mpc.log 2>&1
echo done
