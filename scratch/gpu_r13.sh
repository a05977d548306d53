#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/newton_modes.log
for m in 1 2; do for model in pendulum tvlinear; do timeout 300 python scratch/prof_newton.py $m $model >> gpurun_out/newton_modes.log 2>&1; done; done
echo done
