mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r74_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|Error|assert |^E " gpurun_out/r74_tests.log | head -30
