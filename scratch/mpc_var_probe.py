"""Run-to-run spread of the config-3 MPC leg (bench.mpc_leg): standalone,
then after the bench's e2e leg (host-buffer LQR solves)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import batch as BM
from paper_2409_20027_b200.passes import LqrSolver

orig = BM.BatchSolver.solve_concurrently


def timed(jobs, group=4):
    t0 = time.perf_counter()
    out = orig(jobs, group)
    print(json.dumps({"host_s": round(time.perf_counter() - t0, 3),
                      "launched": [r.launches for r in out]}), flush=True)
    return out


BM.BatchSolver.solve_concurrently = staticmethod(timed)


def mpc(tag):
    out = bench.mpc_leg(torch, P, 1, 0)
    print(json.dumps({"after": tag, "cold_ms": round(out["cold_ms"], 1),
                      "warm_ms": round(out["warm_ms"], 1)}), flush=True)


mpc("nothing")
halves = {}
for system, n in (("pendulum", 32768), ("cartpole", 32768)):
    inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
    solver = LqrSolver(n, bench.T, nx, nu, dtype=torch.float64)
    alpha = bench.lm_alpha_device(torch, solver, inputs, n)
    halves[system] = (solver, inputs, alpha, n, nx, nu)
mpc("inputs")
import gc
for rep in range(2):
    print(bench.e2e_leg(torch, halves, torch.cuda.current_stream(), 1, 5, stacked=False)["value"])
    t0 = time.perf_counter()
    n = gc.collect()
    torch.cuda.synchronize()
    print(json.dumps({"gc_objects": n, "gc_s": round(time.perf_counter() - t0, 3)}), flush=True)
    mpc("e2e+gc")
print(bench.e2e_leg(torch, halves, torch.cuda.current_stream(), 1, 5, stacked=False)["value"])
time.sleep(2.0)
mpc("e2e+sleep2")
