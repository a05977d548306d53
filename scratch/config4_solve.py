"""Config 4 as a full constrained solve on one GPU: barrier method on the
time-varying linearised-quadrotor-like system, T = 2^logT, nx=12, nu=4, |u| <= 2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_20027_b200 as P
logT = int(sys.argv[1]) if len(sys.argv) > 1 else 14
damp = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # A <- damp * A (contractive variant)
T, nx, nu = 1 << logT, 12, 4
rng = np.random.default_rng(20027)
band = np.zeros((nx, nx))
for i in range(4):
    for j in (i, i + 1):
        if j < 4:
            band[3 * i:3 * i + 3, 3 * j:3 * j + 3] = 1.0
A = np.eye(nx)[None] + 0.01 * np.sqrt(0.2) * rng.standard_normal((T, nx, nx)) * band
B = np.sqrt(0.1) * rng.standard_normal((T, nx, nu))
A *= damp
dyn = P.TimeVaryingLinearDynamics(A, B)
qd = rng.uniform(0.1, 10.0, nx)
cost = P.QuadraticCost(np.diag(qd), 0.1 * np.eye(nu), 10 * np.diag(qd))
box = P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
x0 = rng.standard_normal(nx)
P.rollout(dyn, x0, np.zeros((T, nu)))   # warm (library load, solver creation)
torch.cuda.synchronize()
t0 = time.perf_counter()
init = P.rollout(dyn, x0, np.zeros((T, nu)))
torch.cuda.synchronize()
roll_s = time.perf_counter() - t0
t0 = time.perf_counter()
traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init,
                            P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-4,
                                             newton=P.NewtonOptions(max_iters=50)))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print({"T": T, "damp": damp, "rollout_s": round(roll_s, 4), "wall_s": round(wall, 3), "rounds": [r.newton.iterations for r in rep.rounds],
       "terms": [r.newton.termination for r in rep.rounds],
       "max_abs_u": float(np.abs(traj.controls).max()), "cost": rep.rounds[-1].cost})
