mkdir -p gpurun_out
timeout 300 python scratch/prof_long.py 1 > gpurun_out/r80_plain.log 2>&1; echo plain rc=$?; tail -1 gpurun_out/r80_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kw_value_up0|kw_value_down0|kw_prop_down0|kw_value_up\b|kw_value_down\b" --launch-skip 5 --launch-count 5 -o gpurun_out/r80_lqr -f python scratch/prof_long.py 1 > gpurun_out/r80_ncu.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r80_launches.csv python scratch/prof_long.py 1 > /dev/null 2>&1; echo ncu2 rc=$?
