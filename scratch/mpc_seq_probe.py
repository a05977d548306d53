"""Config-3 MPC leg (bench.mpc_leg, every sample printed): the two models'
device loops concurrently on two streams vs one model after the other (each
alone on the whole GPU), fp64 and fp32."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import batch as BM

orig = BM.BatchSolver.solve_concurrently


def seq(jobs, group=16):
    out = []
    for j in jobs:
        out += orig([j], group)
    return out


for mode in sys.argv[1].split(","):
    BM.BatchSolver.solve_concurrently = staticmethod(orig if mode == "conc" else seq)
    for dt in (None, torch.float32):
        for rep in range(2):
            out = bench.mpc_leg(torch, P, 1, 0, dtype=dt)
            print(json.dumps({"mode": mode, "fp32": dt is not None, "cold": out["cold_ms_samples"],
                              "warm": out["warm_ms_samples"]}), flush=True)
