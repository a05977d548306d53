import faulthandler, sys, time
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import DeviceSolver, SolveSettings
from user_models import user_tvlinear, user_pendulum
which = sys.argv[1]
g = np.load("tests/golden/barrier_tvlinear.npz")
if which == "tvl":
    dyn = user_tvlinear(g["A"], g["B"], g["c"])
elif which == "tvl_builtin":
    dyn = P.TimeVaryingLinearDynamics(g["A"], g["B"], g["c"])
nu = dyn.d_u
cost = P.QuadraticCost(g["Q"], 0.1 * np.eye(nu), g["Q"])
init = P.rollout(dyn, g["x0"], g["u0"])
for ex in (sys.argv[2],):
    st = SolveSettings(method=N.METHOD_NEWTON, max_iters=1, hist_cap=1, chunk0=48 if ex == "seq" else 4, chunk=0 if ex == "seq" else 8, rollout=1 if ex == "seq" else 2)
    s = DeviceSolver(dyn, cost, None, 1, st)
    s.load(init.states[None], init.controls[None]); torch.cuda.synchronize(); print("load", flush=True)
    s.expand(); torch.cuda.synchronize(); print("expand", flush=True)
    s.lqr(1.0); torch.cuda.synchronize(); print("lqr", s.read("du")[:4], flush=True)
    s.rollout(); torch.cuda.synchronize(); print("rollout", flush=True)
    s.total_cost(); torch.cuda.synchronize(); print("cost", s.read("cur_cost"), flush=True)
    s.load(init.states[None], init.controls[None])
    s.iterate(1); torch.cuda.synchronize(); print("iterate", s.read("status"), flush=True)
