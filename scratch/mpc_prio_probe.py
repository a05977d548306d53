"""Config-3 MPC leg (bench.mpc_leg) with the two models' device loops on
streams of different priorities: every sample printed."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import batch as BM

orig = BM.BatchSolver.solve_concurrently
for prio in ([0, 0], [-1, 0], [0, -1], [0, 0], [-1, 0], [0, -1]):
    BM.BatchSolver.solve_concurrently = staticmethod(lambda jobs, group=16, p=prio: orig(jobs, group, p))
    for dt in (None, torch.float32):
        out = bench.mpc_leg(torch, P, 1, 0, dtype=dt)
        print(json.dumps({"prio": prio, "fp32": dt is not None, "cold": out["cold_ms_samples"],
                          "warm": out["warm_ms_samples"]}), flush=True)
