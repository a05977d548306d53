mkdir -p gpurun_out
timeout 300 python scratch/prof_mpc.py cartpole > gpurun_out/r61_plain.log 2>&1; echo rc=$?; tail -2 gpurun_out/r61_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_value_fused|k_prop_fused|k_costate_down0|k_rollout|k_cost_partials" --launch-skip 5 --launch-count 5 -o gpurun_out/r61_mpc -f python scratch/prof_mpc.py cartpole > gpurun_out/r61_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/r61_ncu.log
