#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/lqr_plans.log
for args in "12 16" "8 16" "12 12"; do
  echo "== $args" >> gpurun_out/lqr_plans.log
  timeout 120 python scratch/prof_lqr.py $args >> gpurun_out/lqr_plans.log 2>&1
done
timeout 300 python scratch/prof_long.py 3 >> gpurun_out/lqr_plans.log 2>&1
timeout 600 python -m pytest tests/test_gpu_lqr.py tests/test_sharded.py tests/test_gpu_edge.py -q -m gpu >> gpurun_out/lqr_plans.log 2>&1
echo done
