mkdir -p gpurun_out
rm -f gpurun_out/r121_plans.log
for nx in 2 4; do for lt in 8 12 16; do for a in "0 0" "4 4" "4 2" "8 4" "8 2" "16 4" "2 4" "4 16"; do
  echo "== nx$nx T2^$lt $a $(timeout 120 python scratch/prof_lqr.py $nx $lt 20 $a 2>&1 | tr '\n' ' ')" >> gpurun_out/r121_plans.log
done; done; done
for lt in 10 12 14 16; do for a in "0 0" "16 2" "32 4" "32 2" "8 4"; do
  echo "== nx12 T2^$lt $a $(timeout 120 python scratch/prof_lqr.py 12 $lt 10 $a 2>&1 | tr '\n' ' ')" >> gpurun_out/r121_plans.log
done; done
echo done
