"""ncu driver: 3 iterations of the config-3 cart-pole / pendulum batch (32,768 problems)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import BatchSolver
system = sys.argv[1]
n = 32768
probs = bench.models_pkg(P)
bound = 10.0 if system == "cartpole" else 5.0
box = P.BoxConstraint(probs[system].dynamics.d_x, 1, control_lower=-bound, control_upper=bound)
prob = P.ControlProblem(probs[system].dynamics, probs[system].cost, box)
rng = bench.rng_for(0, system)
x0 = bench.initial_states(system, n, rng)
u0 = torch.as_tensor(np.clip(0.1 * bound * rng.standard_normal((n, bench.T, 1)), -0.9 * bound, 0.9 * bound)).cuda()
bs = BatchSolver(prob, n, "barrier", barrier=P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6, newton=P.NewtonOptions(max_iters=50)))
xs = bs.rollout(x0, u0)
bs.solver.load(xs, u0)
bs.solver.iterate(3)
torch.cuda.synchronize()
print("done")
