"""Config 0 (pendulum swing-up, T = 100, batch 1, auto plan): one barrier
solve, for an ncu launch list of the per-iteration kernel sequence."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2409_20027_b200 as P

probs = bench.models_pkg(P)
T0 = 100
rng = np.random.default_rng(20027)
pend = P.ControlProblem(P.PendulumDynamics(T0, P.PendulumParams(damping=0.1, dt=0.05)),
                        probs["pendulum"].cost, probs["pendulum"].constraints)
u0 = np.clip(0.5 * rng.standard_normal((T0, 1)), -4.5, 4.5)
init0 = P.rollout(pend.dynamics, np.array([np.pi, 0.0]), u0)
o0 = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6,
                      newton=P.NewtonOptions(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 50))
try:
    P.barrier_solve(pend, init0, o0)
except Exception as e:  # a capped solve may stall: only the launches matter
    print(type(e).__name__)
