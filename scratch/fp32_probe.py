import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2409_20027_b200 as P
from oracle import pintoc_oracle as O
g = np.load("tests/golden/admm_small.npz")
prob = P.make_swingup_problem("pendulum", 30, 0.05)
d = prob.dynamics.params; c = prob.cost; b = prob.constraints
od = O.Pendulum(gravity=d.gravity, length=d.length, mass=d.mass, damping=d.damping, dt=d.dt)
oc = O.Quadratic(c.Q, c.R, c.Qf, goal=c.x_goal); ob = O.Box(2, 1, control_lower=b.control_lower, control_upper=b.control_upper)
x0, u0 = g["pend_x0"], g["pend_u0"]
u0 = u0.astype(np.float32).astype(float)
xs = O.rollout(od, x0, u0)
z = O.project_box(ob.w(xs, u0)); v = np.zeros_like(z)
r = O.newton_solve(od, oc, ("admm", ob, 1.0, z, v), xs, u0, inner_tol=1e-5)
print("oracle", r.iterations, r.termination)
for h in r.history: print("  ", h)
init = P.rollout(prob.dynamics, x0, u0)
for dt in (torch.float64, torch.float32):
    t, rep = P.newton_solve(prob.dynamics, prob.cost, P.AdmmAugmentation(b, 1.0, z, v), init, P.NewtonOptions(inner_tol=1e-5), dtype=dt)
    print(dt, rep.iterations, rep.termination)
    for h in rep.history: print("  ", (h.cost, h.alpha, h.gain_ratio, h.step_norm, h.accepted))
