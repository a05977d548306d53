"""Per-iteration time of the batched barrier Newton iteration (config-3
halves, 32,768 problems each, T=256, fp64) under scan-tree plans other than
the automatic single sweep: is time-parallelism worth its extra work when
one thread per problem leaves the SMs latency-bound?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import BatchSolver
n = int(os.environ.get("N", "32768"))
plans = [(0, 0), (64, 4), (32, 8), (16, 16), (32, 4), (16, 4)]
for system in ("pendulum", "cartpole"):
    probs = bench.models_pkg(P)
    bound = 10.0 if system == "cartpole" else 5.0
    box = P.BoxConstraint(probs[system].dynamics.d_x, 1, control_lower=-bound, control_upper=bound)
    prob = P.ControlProblem(probs[system].dynamics, probs[system].cost, box)
    rng = bench.rng_for(0, system)
    x0 = bench.initial_states(system, n, rng)
    u0 = torch.as_tensor(np.clip(0.1 * bound * rng.standard_normal((n, bench.T, 1)), -0.9 * bound, 0.9 * bound)).cuda()
    for ex in ("auto", "parallel"):
        for c0, c1 in plans:
            if ex == "parallel" and c0 == 0:
                continue
            opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6,
                                    newton=P.NewtonOptions(max_iters=50, executor=ex))
            bs = BatchSolver(prob, n, "barrier", barrier=opts, chunk0=c0, chunk=c1)
            xs = bs.rollout(x0, u0)
            s = bs.solver
            times = []
            for rep in range(2):
                s.load(xs, u0)
                s.iterate(2)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); s.iterate(10); b.record(); torch.cuda.synchronize()
                times.append(a.elapsed_time(b) / 10)
            print(system, n, ex, (c0, c1), "ms/iteration", [round(t, 3) for t in times], flush=True)
            del bs, s
