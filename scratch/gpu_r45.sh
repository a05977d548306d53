set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_newton.py tests/test_gpu_edge.py tests/test_gpu_newton.py tests/test_gpu_passes.py -x -q > gpurun_out/r45_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r45_tests.log
timeout 300 python scratch/config4_solve.py 18 > gpurun_out/r45_c18.log 2>&1; echo c18 rc=$?
cat gpurun_out/r45_c18.log | tail -3
timeout 300 python scratch/config4_solve.py 20 > gpurun_out/r45_c20.log 2>&1; echo c20 rc=$?
cat gpurun_out/r45_c20.log | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r45_c18_launches.csv python scratch/config4_solve.py 18 > gpurun_out/r45_ncu.log 2>&1; echo ncu rc=$?
