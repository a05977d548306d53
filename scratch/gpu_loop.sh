# device-resident solve loop (ptc_solver_loop): parity test, then the MPC /
# single-solve legs with the device loop and with the host-polled loop
timeout 600 python -m pytest tests/test_gpu_edge.py -x -q -p no:cacheprovider -k "device_loop or concurrent" > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/s2_pytest.log
X="--no-cpu-baseline --no-e2e --no-sweep --no-newton-sweep --no-long --no-c4solve"
timeout 600 python bench.py $X > gpurun_out/s2_dev.log 2>&1; echo "dev rc $?"
PTC_HOST_LOOP=1 timeout 600 python bench.py $X > gpurun_out/s2_host.log 2>&1; echo "host rc $?"
timeout 600 python bench.py $X > gpurun_out/s2_dev2.log 2>&1; echo "dev2 rc $?"
for f in s2_dev s2_host s2_dev2; do python - "$f" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/"+sys.argv[1]+".log").read().strip().splitlines()[-1])
m=d.get("mpc_config3",{}); m32=d.get("mpc_config3_fp32",{}); s=d.get("single_solves",{})
print(sys.argv[1], "mpc cold", m.get("cold_ms_samples"), "warm", m.get("warm_ms_samples"), "fp32 warm", m32.get("warm_ms_samples"), "c0", s.get("config0",{}).get("gpu_s"), "c2", s.get("config2",{}).get("gpu_s"))
PY
done
