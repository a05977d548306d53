#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/cfg4solve.log
for l in 12 16 20; do timeout 600 python scratch/config4_solve.py $l >> gpurun_out/cfg4solve.log 2>&1; done
echo done
