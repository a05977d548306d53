mkdir -p gpurun_out
timeout 300 python scratch/prof_newton.py 2 tvlinear > gpurun_out/r130_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r130_newton.csv python scratch/prof_newton.py 2 tvlinear > gpurun_out/r130_ncu.log 2>&1; echo ncu rc=$?
