"""Active-set profile of the config-3 MPC solve: per group of 4 device
iterations, the number of problems still running and the ms per iteration
(cold solve, one model at a time, 32,768 problems, fp64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200 import BatchSolver

n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
for system in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("pendulum", "cartpole")):
    probs = bench.models_pkg(P)
    bound = 10.0 if system == "cartpole" else 5.0
    box = P.BoxConstraint(probs[system].dynamics.d_x, 1, control_lower=-bound, control_upper=bound)
    prob = P.ControlProblem(probs[system].dynamics, probs[system].cost, box)
    rng = bench.rng_for(0, system)
    x0 = bench.initial_states(system, n, rng)
    u0 = torch.as_tensor(np.clip(0.1 * bound * rng.standard_normal((n, bench.T, 1)),
                                 -0.9 * bound, 0.9 * bound)).cuda()
    opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6, newton=P.NewtonOptions(max_iters=50))
    bs = BatchSolver(prob, n, "barrier", barrier=opts)
    xs = bs.rollout(x0, u0)
    s = bs.solver
    s.load(xs, u0)
    s.iterate(1)
    torch.cuda.synchronize()
    rows, it, total = [], 1, 0.0
    while True:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.iterate(4); b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        total += ms
        r = s.running()
        rows.append((it, r, ms / 4))
        it += 4
        if r == 0 or it > 480:
            break
    print(system, "total ms", round(total, 1), flush=True)
    for k in range(0, len(rows), 4):
        i, r, m = rows[k]
        print(f"  it {i:4d} running {r:6d} ms/it {m:.3f}")
    buckets = {}
    for i, r, m in rows:
        key = "32768" if r >= 16384 else ">=4096" if r >= 4096 else ">=512" if r >= 512 else "<512"
        buckets.setdefault(key, [0, 0.0])
        buckets[key][0] += 4
        buckets[key][1] += 4 * m
    print("  by active set:", {k: (v[0], round(v[1], 1)) for k, v in buckets.items()}, flush=True)
