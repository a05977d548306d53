#!/bin/bash
mkdir -p gpurun_out
for args in "12 16" "12 16 3 16 8" "12 16 3 8 4" "12 16 3 32 8" "8 16" "12 12" "12 8"; do
  echo "== $args" >> gpurun_out/lqr_plans.log
  timeout 120 python scratch/prof_lqr.py $args >> gpurun_out/lqr_plans.log 2>&1
done
PTC_NO_GRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lqr12.csv python scratch/prof_lqr.py 12 16 1 > gpurun_out/ncu_lqr12.log 2>&1
echo done
