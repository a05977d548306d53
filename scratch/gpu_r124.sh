mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^kw_value_(up|down)$" --launch-skip 12 --launch-count 4 -o gpurun_out/r124_tree -f python scratch/prof_long.py 1 > gpurun_out/r124_ncu.log 2>&1; echo ncu rc=$?
