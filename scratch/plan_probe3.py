"""LQR-scan solve per half at strong-scaling batch sizes: single sweep
(chunk0 = T) vs the auto plan (blocked tree below 16,384 problems)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
out = {}
for system in ("pendulum", "cartpole"):
    full, nx, nu = bench.build_inputs(P, torch, system, 32768, 0)
    for n in (32768, 16384):
        ins = [t[:, :, :n].contiguous() for t in full]
        for name, (c0, c1) in (("sweep", (bench.T, 0)), ("k128", (128, 8)), ("k64", (64, 8)),
                               ("k32", (32, 8))):
            s = LqrSolver(n, bench.T, nx, nu, chunk0=c0, chunk=c1)
            alpha = torch.full((n,), 64.0, dtype=torch.float64, device="cuda")
            for _ in range(3): s.solve(*ins, alpha)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20): s.solve(*ins, alpha)
            b.record(); torch.cuda.synchronize()
            out[f"{system}_{n}_{name}"] = (round(a.elapsed_time(b) / 20, 4), s.plan())
            del s
print(json.dumps(out))
