mkdir -p gpurun_out
timeout 900 python scratch/plan_probe.py > gpurun_out/r64_plans.log 2>&1; echo rc=$?
cat gpurun_out/r64_plans.log | tail -10
