import faulthandler, sys, time
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2409_20027_b200 as P
from user_models import user_tvlinear
t0 = time.time()
g = np.load("tests/golden/barrier_tvlinear.npz")
dyn = user_tvlinear(g["A"], g["B"], g["c"])
nu = dyn.d_u
cost = P.QuadraticCost(g["Q"], 0.1 * np.eye(nu), g["Q"])
box = P.BoxConstraint(dyn.d_x, nu, control_lower=-2.0, control_upper=2.0)
init = P.rollout(dyn, g["x0"], g["u0"])
print("rollout", time.time() - t0, flush=True)
traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(max_iters=3, executor="sequential"))
print("newton", rep.iterations, rep.termination, time.time() - t0, flush=True)
traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init,
                            P.BarrierOptions(newton=P.NewtonOptions(executor="sequential")))
print("barrier", [r.newton.iterations for r in rep.rounds], list(g["sol_round_iters"]), time.time() - t0, flush=True)
