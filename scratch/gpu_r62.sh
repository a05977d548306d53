mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python scratch/prof_mpc.py cartpole; done > gpurun_out/r62_plain.log 2>&1; cat gpurun_out/r62_plain.log | grep ms
for i in 1 2; do timeout 300 python scratch/prof_mpc.py pendulum; done >> gpurun_out/r62_plain.log 2>&1; grep ms gpurun_out/r62_plain.log | tail -2
timeout 900 python -m pytest tests/test_gpu_newton.py tests/test_gpu_harness.py tests/test_gpu_edge.py tests/test_gpu_passes.py -x -q > gpurun_out/r62_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r62_tests.log
