mkdir -p gpurun_out
timeout 600 python scratch/config4_solve.py 20 0.9999 > gpurun_out/r127_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r127_c4.csv python scratch/config4_solve.py 20 0.9999 > gpurun_out/r127_ncu.log 2>&1; echo ncu rc=$?
