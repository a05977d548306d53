"""Batch-1 pendulum barrier solve (config 0 shape) per scan plan (K0, K):
ms per Newton iteration, iteration counts."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import BatchSolver

probs = bench.models_pkg(P)
for T0 in (100, 256, 1024):
    rng = np.random.default_rng(20027)
    pend = P.ControlProblem(P.PendulumDynamics(T0, P.PendulumParams(damping=0.1, dt=0.05)),
                            probs["pendulum"].cost, probs["pendulum"].constraints)
    u0 = torch.as_tensor(np.clip(0.5 * rng.standard_normal((1, T0, 1)), -4.5, 4.5))
    o0 = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6)
    plans = [(0, 0), (4, 4), (4, 8), (8, 4), (8, 8), (10, 10), (16, 8), (16, 16), (32, 8), (T0, 0)]
    for c0, c1 in plans:
        if c0 > T0:
            continue
        bs = BatchSolver(pend, 1, "barrier", barrier=o0, chunk0=c0, chunk=c1)
        xs = bs.rollout(np.array([[np.pi, 0.0]]), u0)
        r = bs.solve(xs, u0)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            r = bs.solve(xs, u0)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        it = int(r.round_iters.sum())
        print(json.dumps({"T": T0, "plan": [c0, c1], "s": round(min(ts), 4), "iters": it,
                          "ms_per_iter": round(1e3 * min(ts) / max(it, 1), 4),
                          "status": int(r.status[0])}), flush=True)
