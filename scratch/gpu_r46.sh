set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_newton.py tests/test_gpu_edge.py tests/test_gpu_newton.py tests/test_gpu_passes.py tests/test_gpu_harness.py -x -q > gpurun_out/r46_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r46_tests.log
timeout 300 python scratch/config4_solve.py 18 > gpurun_out/r46_c18.log 2>&1; echo c18 rc=$?
tail -1 gpurun_out/r46_c18.log
timeout 300 python scratch/config4_solve.py 20 0.9999 > gpurun_out/r46_c20.log 2>&1; echo c20 rc=$?
tail -1 gpurun_out/r46_c20.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r46_c20_launches.csv python scratch/config4_solve.py 20 0.9999 > gpurun_out/r46_ncu.log 2>&1; echo ncu rc=$?
