"""LQR latency at batch 1 (config 1 inputs) for nx 2 / 4: thread-per-unit
kernels vs the warp-per-unit kernels (PTC_WIDE_SMALL=1)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2409_20027_b200.passes import LqrSolver
out = {}
for nx in (2, 4):
    nu = nx // 2
    row = {}
    for logT in (8, 10, 12, 14, 16):
        Tn = 1 << logT
        e = bench.config1_inputs(np.random.default_rng([1, nx, logT]), Tn, nx, nu)
        dev = torch.device("cuda")
        soa = lambda a: torch.as_tensor(a.reshape(a.shape[0], -1).T.copy()).unsqueeze(-1).to(dev)
        ins = [soa(e[k]) for k in ("P", "R", "M", "d", "Fx", "Fu", "PT")]
        alpha = torch.zeros(1, dtype=torch.float64, device=dev)
        s = LqrSolver(1, Tn, nx, nu)
        for _ in range(3):
            s.solve(*ins, alpha)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            s.solve(*ins, alpha)
        b.record()
        torch.cuda.synchronize()
        row[Tn] = round(a.elapsed_time(b) / 10, 4)
        if logT == 10:
            row["du_checksum"] = float(s.du.abs().sum())
    out[f"nx{nx}"] = row
print(os.environ.get("PTC_WIDE_SMALL", "0"), json.dumps(out))
