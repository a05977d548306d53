mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r108_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r108_tests.log; grep -E "FAILED|^E " gpurun_out/r108_tests.log | head
