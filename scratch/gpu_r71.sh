mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_newton.py -q -k fp32 > gpurun_out/r71_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|Error|assert |^E " gpurun_out/r71_tests.log | head -20
