mkdir -p gpurun_out
timeout 1200 python scratch/plan_probe2.py > gpurun_out/r65_plans.log 2>&1; echo rc=$?
cat gpurun_out/r65_plans.log | tail -6
