mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kwn_costate_down0|kwn_costate_up0|kwn_roll_up0|kwn_roll_down0|kw_value_up0|kw_value_down0" --launch-skip 10 --launch-count 6 -o gpurun_out/r58_c4 -f python scratch/config4_solve.py 18 > gpurun_out/r58_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/r58_ncu.log
