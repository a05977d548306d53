"""Rank 0's share of an 8-GPU headline run (8,192 problems) on one GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
bp, bc = bench.half_sizes(bench.B_TOTAL // world)
halves = {}
for system, n in (("pendulum", bp), ("cartpole", bc)):
    inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
    sol = LqrSolver(n, bench.T, nx, nu)
    alpha = bench.lm_alpha_device(torch, sol, inputs, n)
    halves[system] = (sol, inputs, alpha)
torch.cuda.synchronize()
for _ in range(5):
    for sol, ins, al in halves.values():
        sol.solve(*ins, al)
torch.cuda.synchronize()
print("plan", halves["cartpole"][0].plan())
