mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r94_c20_launches.csv python scratch/config4_solve.py 20 0.9999 > gpurun_out/r94_ncu.log 2>&1; echo ncu rc=$?
