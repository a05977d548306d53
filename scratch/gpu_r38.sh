#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/cfg4solve.log gpurun_out/newton_modes.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for l in 12 16; do timeout 600 python scratch/config4_solve.py $l >> gpurun_out/cfg4solve.log 2>&1; done
for m in 2; do for model in pendulum tvlinear; do timeout 300 python scratch/prof_newton.py $m $model >> gpurun_out/newton_modes.log 2>&1; done; done
echo done
