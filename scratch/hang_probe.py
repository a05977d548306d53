import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import DeviceSolver, SolveSettings
for logT in (10, 14):
    Tn = 1 << logT
    rng = np.random.default_rng([3, logT])
    dyn = P.PendulumDynamics(Tn, P.PendulumParams(damping=1.0, dt=0.05))
    hang = np.array([0.0, 0.0])
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]), x_goal=hang)
    x0 = hang + np.array([0.5, 0.0]); us = 0.02 * rng.standard_normal((1, Tn, 1))
    for ex, ch in (("par", (4, 8)), ("auto", (0, 0))):
        s = DeviceSolver(dyn, cost, None, 1, SolveSettings(method=N.METHOD_NEWTON, max_iters=1000, inner_tol=1e-300, hist_cap=32, chunk0=ch[0], chunk=ch[1], rollout=2 if ex == "par" else 0))
        X = torch.zeros(1, Tn + 1, 2, dtype=torch.float64); X[0, 0] = torch.as_tensor(x0)
        s.load(X, torch.as_tensor(us)); s.rollout(); X = s.field("states", Tn + 1, (2,)).contiguous()
        s.load(X, torch.as_tensor(us)); s.iterate(10); torch.cuda.synchronize()
        h = s.history()[:10, :, 0].cpu().numpy()
        print(Tn, ex, "status", int(s.read("status")[0]), "rollout_state", int(s.read("rollout_state")[0]))
        for r in h: print("   ", np.round(r, 6))
