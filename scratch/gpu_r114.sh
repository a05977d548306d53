mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kw_value_up0|kw_value_down0" --launch-skip 4 --launch-count 2 -o gpurun_out/r114_lqr -f python scratch/prof_long.py 1 > gpurun_out/r114_ncu.log 2>&1; echo ncu rc=$?
