"""Newton-iteration latency sweep (batch 1) by rollout mode: args mode [model].

model "pendulum": swing-up from random controls, timed after 12 settling
iterations; "tvlinear": config-1 style random time-varying system (nx=4,
nu=2) with the quadratic cost, timed after its first (exact) iteration.
Prints ms per iteration, how many of the 4 timed iterations did full work
(finite step norm), and the rollout state of the last one.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, statistics
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import DeviceSolver, SolveSettings

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
model = sys.argv[2] if len(sys.argv) > 2 else "pendulum"
out = {}
for logT in (8, 10, 12, 14, 16):
    Tn = 1 << logT
    rng = np.random.default_rng([3, logT])
    if model == "pendulum":
        dyn = P.PendulumDynamics(Tn, P.PendulumParams(damping=0.1, dt=0.05))
        cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
        nx, nu, settle = 2, 1, 12
        x0 = np.array([np.pi, 0.0])
        us = 0.5 * rng.standard_normal((1, Tn, 1))
    else:
        nx, nu, settle = 4, 2, 2
        A = np.eye(nx)[None] + 0.05 * rng.standard_normal((Tn, nx, nx))
        A *= np.minimum(1.0, 1.0 / np.max(np.abs(np.linalg.eigvals(A)), axis=1))[:, None, None]
        Bm = np.sqrt(0.1) * rng.standard_normal((Tn, nx, nu))
        dyn = P.TimeVaryingLinearDynamics(A, Bm, 0.1 * rng.standard_normal((Tn, nx)))
        cost = P.QuadraticCost(np.eye(nx), 0.1 * np.eye(nu), 10 * np.eye(nx))
        x0 = rng.standard_normal(nx)
        us = 0.1 * rng.standard_normal((1, Tn, nu))
    s = DeviceSolver(dyn, cost, None, 1, SolveSettings(method=N.METHOD_NEWTON, max_iters=1000,
                                                        inner_tol=1e-300, rollout=mode,
                                                        hist_cap=32))
    us = torch.as_tensor(us)
    X = torch.zeros(1, Tn + 1, nx, dtype=torch.float64)
    X[0, 0] = torch.as_tensor(x0)
    s.load(X, us)
    s.rollout()
    X = s.field("states", Tn + 1, (nx,)).contiguous()
    per, full = [], []
    for _ in range(3):
        s.load(X, us)
        s.iterate(settle)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.iterate(4)
        b.record()
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b) / 4)
        h = s.history()[:, :, 0].cpu().numpy()[settle:settle + 4]
        full.append((int(np.isfinite(h[:, 3]).sum()), int(s.read("rollout_state")[0])))
    out[Tn] = (round(statistics.median(per), 4), full)
print(json.dumps({"mode": mode, "model": model, "ms_per_iteration": out}))
