#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/lqr_plans.log gpurun_out/mpc.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for args in "12 16" "8 16" "12 12"; do
  echo "== $args" >> gpurun_out/lqr_plans.log
  timeout 120 python scratch/prof_lqr.py $args >> gpurun_out/lqr_plans.log 2>&1
done
timeout 300 python scratch/prof_long.py 3 >> gpurun_out/lqr_plans.log 2>&1
timeout 900 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench, paper_2409_20027_b200 as P
print(json.dumps(bench.mpc_leg(torch, P, 1, 0)))" > gpurun_out/mpc.log 2>&1
echo done
