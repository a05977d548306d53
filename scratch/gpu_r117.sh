mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lqr.py tests/test_gpu_wide_newton.py tests/test_gpu_fullsize.py tests/test_gpu_elements.py -m gpu -q -x > gpurun_out/r117_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r117_tests.log; grep -E "^E " gpurun_out/r117_tests.log | head -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kw_value_up0|kw_value_down0" --launch-skip 4 --launch-count 2 -o gpurun_out/r117_lqr -f python scratch/prof_long.py 1 > gpurun_out/r117_ncu.log 2>&1; echo ncu rc=$?
