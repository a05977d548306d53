#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/newton_modes.log
for m in 1 2 0; do timeout 300 python scratch/prof_newton.py $m >> gpurun_out/newton_modes.log 2>&1; done
echo done
