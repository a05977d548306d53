#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep --no-newton-sweep --no-long --no-mpc > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo "rc=$?" >> gpurun_out/bench_fp32.err
echo done
