import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import golden, rel_gap
import paper_2409_20027_b200 as P
from oracle import pintoc_oracle as O
g = golden("newton_lq")
for i in range(int(g["count"])):
    p = f"{i}_"
    n, du = g[p + "us"].shape
    dyn = P.LinearDynamics(g[p + "A"], g[p + "B"], horizon=n)
    cost = P.QuadraticCost(g[p + "Q"], g[p + "R"], g[p + "Qf"], x_goal=g[p + "goal"])
    init = P.rollout(dyn, g[p + "x0"], np.zeros((n, du)))
    a0 = float(g[p + "alpha0"])
    traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(alpha0=a0))
    h = np.array([(r.cost, r.alpha, r.gain_ratio, r.step_norm, r.accepted) for r in rep.history])
    ref = g[p + "hist"]
    print(i, n, g[p+"A"].shape, du, a0, rep.termination, len(h), len(ref), "u gap", rel_gap(traj.controls, g[p+"us"]))
    np.set_printoptions(precision=17, linewidth=200)
    for k in range(min(len(h), len(ref))):
        print("   ", k, h[k], ref[k])
