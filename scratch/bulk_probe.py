"""LQR-scan solve time per config-3 half: TMA ring (bulk_sweeps.cuh) vs
register path (PTC_BULK=0), fp64 / fp32; run once per PTC_BULK setting."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
out = {}
for system in ("pendulum", "cartpole"):
    inputs, nx, nu = bench.build_inputs(P, torch, system, 32768, 0)
    for dt in (torch.float64, torch.float32):
        ins = [t.to(dt) for t in inputs]
        s = LqrSolver(32768, bench.T, nx, nu, dtype=dt)
        alpha = torch.full((32768,), 64.0, dtype=torch.float64, device="cuda")
        for _ in range(3): s.solve(*ins, alpha)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): s.solve(*ins, alpha)
        b.record(); torch.cuda.synchronize()
        out[f"{system}_{str(dt)[-7:]}"] = round(a.elapsed_time(b) / 20, 4)
        del s, ins
    del inputs
print(os.environ.get("PTC_BULK", "auto"), json.dumps(out))
