mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_newton.py -x -q > gpurun_out/r59_tests.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/r59_tests.log
