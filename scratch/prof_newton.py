"""Newton-iteration latency sweep (pendulum, batch 1) for rollout modes: args [mode]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, statistics
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import DeviceSolver, SolveSettings
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
out = {}
for logT in (8, 10, 12, 14, 16):
    Tn = 1 << logT
    dyn = P.PendulumDynamics(Tn, P.PendulumParams(damping=0.1, dt=0.05))
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    s = DeviceSolver(dyn, cost, None, 1, SolveSettings(method=N.METHOD_NEWTON, max_iters=1000,
                                                        inner_tol=1e-300, rollout=mode,
                                                        hist_cap=32))
    rng = np.random.default_rng([3, logT])
    us = torch.as_tensor(0.5 * rng.standard_normal((1, Tn, 1)))
    X = torch.zeros(1, Tn + 1, 2, dtype=torch.float64)
    X[0, 0, 0] = np.pi
    s.load(X, us)
    s.rollout()
    X = s.field("states", Tn + 1, (2,)).contiguous()
    per, full = [], []
    for _ in range(3):
        s.load(X, us)
        s.iterate(12)  # let the LM weight settle on solvable subproblems
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.iterate(4)
        b.record()
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b) / 4)
        h = s.history()[:, :, 0].cpu().numpy()[12:16]
        full.append(int(np.isfinite(h[:, 3]).sum()))
    out[Tn] = (round(statistics.median(per), 4), full)
print(json.dumps({"mode": mode, "ms_per_iteration(full-work iterations of 4)": out}))
