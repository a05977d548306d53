#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edge.py -q > gpurun_out/pytest_edge.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_edge.log
timeout 900 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench, paper_2409_20027_b200 as P
print(json.dumps(bench.mpc_leg(torch, P, 1, 0)))" > gpurun_out/mpc.log 2>&1
echo done
