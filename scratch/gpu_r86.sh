mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r86_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r86_tests.log
