set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s1_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/s1_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s1_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/s1_bench.log 2>&1; echo "bench rc $?"
tail -1 gpurun_out/s1_bench.log
