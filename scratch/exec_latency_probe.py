"""Batch-1 barrier solves (config 0's pendulum swing-up and longer horizons)
per executor: device seconds per solve and per Newton iteration."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, paper_2409_20027_b200 as P

probs = bench.models_pkg(P)
for T0 in (100, 256, 1024):
    rng = np.random.default_rng(20027)
    pend = P.ControlProblem(P.PendulumDynamics(T0, P.PendulumParams(damping=0.1, dt=0.05)),
                            probs["pendulum"].cost, probs["pendulum"].constraints)
    u0 = np.clip(0.5 * rng.standard_normal((T0, 1)), -4.5, 4.5)
    init0 = P.rollout(pend.dynamics, np.array([np.pi, 0.0]), u0)
    for ex in (P.SEQUENTIAL, P.AUTO, P.PARALLEL):
        o0 = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6, newton=P.NewtonOptions(executor=ex))
        P.barrier_solve(pend, init0, o0)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            _, rep = P.barrier_solve(pend, init0, o0)
            ts.append(time.perf_counter() - t)
        it = sum(r.newton.iterations for r in rep.rounds)
        print(json.dumps({"T": T0, "executor": ex, "s": round(min(ts), 4), "iters": it,
                          "ms_per_iter": round(1e3 * min(ts) / it, 4)}), flush=True)
