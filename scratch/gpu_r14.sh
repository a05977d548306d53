#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/newton_modes.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 1 2; do for model in pendulum tvlinear; do timeout 300 python scratch/prof_newton.py $m $model >> gpurun_out/newton_modes.log 2>&1; done; done
echo done
