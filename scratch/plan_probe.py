"""Scan-plan sweep for the config-3 LQR solve at per-GPU batch sizes of the
strong-scaling runs (65,536 / N problems per GPU, half per model)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
T = bench.T
plans = [(T, 0), (4, 8), (8, 8), (16, 8), (32, 8), (64, 8), (8, 4), (16, 4), (32, 4), (16, 16),
         (32, 16), (64, 16), (128, 2)]
res = {}
for n in (2048, 4096, 8192, 16384):
    for system in ("pendulum", "cartpole"):
        inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
        base = LqrSolver(n, T, nx, nu)
        alpha = bench.lm_alpha_device(torch, base, inputs, n)
        row = {}
        for c0, c1 in plans:
            s = LqrSolver(n, T, nx, nu, chunk0=c0, chunk=c1)
            for _ in range(3):
                s.solve(*inputs, alpha)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                s.solve(*inputs, alpha)
            b.record()
            torch.cuda.synchronize()
            row[f"{c0}/{c1}"] = round(a.elapsed_time(b) / 10, 4)
            del s
        auto = LqrSolver(n, T, nx, nu).plan()
        res[f"{system}_{n}"] = {"auto": auto, "ms": row,
                                "best": min(row, key=row.get)}
        print(json.dumps({f"{system}_{n}": res[f"{system}_{n}"]}), flush=True)
        del inputs, base
        torch.cuda.empty_cache()
