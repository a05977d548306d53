#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-newton-sweep --no-mpc > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo "rc=$?" >> gpurun_out/torchrun1.err
CMD="python scratch/prof_mpc.py cartpole"
timeout 300 $CMD > gpurun_out/plain_mpc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_value_fused|k_prop_fused|k_costate_down0|k_rollout|k_cost_partials" -s 5 -c 5 -o gpurun_out/prof_mpc $CMD > gpurun_out/ncu_mpc.log 2>&1
CMD2="python scratch/prof_long.py 1"
timeout 300 $CMD2 > gpurun_out/plain_long.log 2>&1 && \
PTC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_long.csv $CMD2 > gpurun_out/ncu_launch_long.log 2>&1
echo done
