"""ncu driver: batch-1 Newton iterations of the time-varying linear model
(bench.newton_latency_sweep's tvlinear, nx 4, nu 2) at horizon 2^logT:
2 settling iterations, then 1 iteration to profile (PTC_NO_GRAPH=1 under
ncu keeps every launch visible)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import DeviceSolver, SolveSettings
logT = int(sys.argv[1]) if len(sys.argv) > 1 else 8
Tn = 1 << logT
rng = np.random.default_rng([3, logT])
nx, nu = 4, 2
A = np.eye(nx)[None] + 0.05 * rng.standard_normal((Tn, nx, nx))
A *= np.minimum(1.0, 1.0 / np.max(np.abs(np.linalg.eigvals(A)), axis=1))[:, None, None]
Bm = np.sqrt(0.1) * rng.standard_normal((Tn, nx, nu))
dyn = P.TimeVaryingLinearDynamics(A, Bm, 0.1 * rng.standard_normal((Tn, nx)))
cost = P.QuadraticCost(np.eye(nx), 0.1 * np.eye(nu), 10 * np.eye(nx))
s = DeviceSolver(dyn, cost, None, 1, SolveSettings(method=N.METHOD_NEWTON, max_iters=1000,
                                                    inner_tol=1e-300, hist_cap=32))
us = torch.as_tensor(0.1 * rng.standard_normal((1, Tn, nu)))
X = torch.zeros(1, Tn + 1, nx, dtype=torch.float64)
X[0, 0] = torch.as_tensor(rng.standard_normal(nx))
s.load(X, us)
s.rollout()
X = s.field("states", Tn + 1, (nx,)).contiguous()
s.load(X, us)
s.iterate(2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.iterate(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
