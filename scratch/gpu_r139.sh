mkdir -p gpurun_out
timeout 300 python scratch/prof_lqr.py 12 16 3 > gpurun_out/r139_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r139_lqr12.csv python scratch/prof_lqr.py 12 16 3 > gpurun_out/r139_ncu.log 2>&1; echo ncu rc=$?
