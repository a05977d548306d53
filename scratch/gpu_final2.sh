# final check after the priority / mixed-loop changes: GPU suite, smoke, default bench
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g_pytest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/g_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1; echo "bench rc $?"
