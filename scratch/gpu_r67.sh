mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_behaviour.py -q > gpurun_out/r67_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|Error|assert" gpurun_out/r67_tests.log | head -30
