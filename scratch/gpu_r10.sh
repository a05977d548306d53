#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 1 2 0; do timeout 300 python scratch/prof_newton.py $m >> gpurun_out/newton_modes.log 2>&1; done
echo done
