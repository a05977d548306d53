mkdir -p gpurun_out
rm -f gpurun_out/r119_long.log gpurun_out/r119_lqr12.log
for a in "128 8" "128 4" "128 2" "256 4" "256 2" "64 4" "64 2"; do timeout 300 python scratch/prof_long.py 3 $a >> gpurun_out/r119_long.log 2>&1; done
for a in "0 0" "8 4" "8 2" "16 4" "16 2" "4 4" "4 2"; do echo "== $a" >> gpurun_out/r119_lqr12.log; timeout 300 python scratch/prof_lqr.py 12 16 5 $a >> gpurun_out/r119_lqr12.log 2>&1; done
for a in "0 0" "8 4" "8 2" "16 2"; do echo "== 10: $a" >> gpurun_out/r119_lqr12.log; timeout 300 python scratch/prof_lqr.py 12 10 5 $a >> gpurun_out/r119_lqr12.log 2>&1; done
echo done
