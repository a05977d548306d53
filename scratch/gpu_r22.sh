#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/lqr_plans.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for args in "12 16" "12 16 3 8 8" "12 16 3 16 8" "8 16" "8 16 3 8 8" "12 12" "12 8" "8 8"; do
  echo "== $args" >> gpurun_out/lqr_plans.log
  timeout 120 python scratch/prof_lqr.py $args >> gpurun_out/lqr_plans.log 2>&1
done
timeout 300 python scratch/prof_long.py 3 >> gpurun_out/lqr_plans.log 2>&1
echo done
