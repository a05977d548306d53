mkdir -p gpurun_out
for bs in 128 64 32 0; do
  PTC_LQR_BLOCK=$bs timeout 600 python scratch/shard_probe_blk.py > gpurun_out/r118_blk$bs.json 2> gpurun_out/r118_blk$bs.err; echo bs=$bs rc=$?
done
timeout 600 python -m pytest tests/test_gpu_lqr.py tests/test_gpu_newton.py -m gpu -q -x > gpurun_out/r118_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r118_tests.log
