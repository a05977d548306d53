"""Run-to-run spread of the config-3 MPC leg (bench.mpc_leg, median of 3
solves per leg, every sample printed) for host poll groups of 4 / 16
device iterations."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import batch as BM

orig = BM.BatchSolver.solve_concurrently
for group in [int(g) for g in (sys.argv[1] if len(sys.argv) > 1 else "4,16").split(",")]:
    BM.BatchSolver.solve_concurrently = staticmethod(lambda jobs, g=group: orig(jobs, g))
    for rep in range(2):
        out = bench.mpc_leg(torch, P, 1, 0)
        print(json.dumps({"group": group, "cold": out["cold_ms_samples"],
                          "warm": out["warm_ms_samples"]}), flush=True)
