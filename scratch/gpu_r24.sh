#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/long_plans.log
for a in "4 8" "8 8" "16 8" "32 8" "4 16" "2 8"; do timeout 300 python scratch/prof_long.py 3 $a >> gpurun_out/long_plans.log 2>&1; done
echo done
