mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kw_value_up0" --launch-skip 2 --launch-count 1 -o gpurun_out/r87_up0 -f python scratch/prof_long.py 1 > gpurun_out/r87_ncu.log 2>&1; echo ncu rc=$?
