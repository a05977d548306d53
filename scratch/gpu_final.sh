# round-end check of the session's code: GPU suite, smoke, default bench,
# launch list of the headline step (ncu, after the plain runs exit 0)
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/f_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo "bench rc $?"
X="--no-cpu-baseline --no-e2e --no-sweep --no-newton-sweep --no-long --no-mpc --no-fp32 --no-c4solve --no-solves"
timeout 600 python bench.py --steps 2 --warmup 3 $X > gpurun_out/f_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 $X > gpurun_out/f_ncu.log 2>&1; echo "ncu rc $?"
