mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_newton.py -x -q > gpurun_out/r52_tests.log 2>&1; echo tests rc=$?
tail -40 gpurun_out/r52_tests.log
