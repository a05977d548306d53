#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/long_plans.log
for a in "32 8" "64 8" "128 8" "64 16" "32 16" "256 8"; do timeout 300 python scratch/prof_long.py 3 $a >> gpurun_out/long_plans.log 2>&1; done
echo done
