"""Profile driver: a short batched barrier solve of the config-3 cart-pole half (32,768 problems)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import BatchSolver
n = 32768
system = sys.argv[1] if len(sys.argv) > 1 else "cartpole"
probs = bench.models_pkg(P)
bound = 10.0 if system == "cartpole" else 5.0
box = P.BoxConstraint(probs[system].dynamics.d_x, 1, control_lower=-bound, control_upper=bound)
prob = P.ControlProblem(probs[system].dynamics, probs[system].cost, box)
rng = bench.rng_for(0, system)
x0 = bench.initial_states(system, n, rng)
u0 = np.clip(0.1 * bound * rng.standard_normal((n, bench.T, 1)), -0.9 * bound, 0.9 * bound)
opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=0.05, newton=P.NewtonOptions(max_iters=6))
bs = BatchSolver(prob, n, "barrier", barrier=opts)
xs = bs.rollout(x0, torch.as_tensor(u0))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
res = bs.solve(xs, torch.as_tensor(u0).cuda())
b.record()
torch.cuda.synchronize()
print("ms", a.elapsed_time(b), "launches", res.launches, "iters", int(res.inner_iterations.sum()))
