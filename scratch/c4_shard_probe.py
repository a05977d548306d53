"""Strong-scaling projection of the time-sharded config-4 barrier solve:
N ranks emulated on one B200 (phases of all ranks run back to back, gathers
become stacks), total device time / N = one rank's share without the
NVLink collectives (8 all-gathers of <= 456 words and 3 small all-reduces
per iteration)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import SolveSettings
from paper_2409_20027_b200.sharded import BlockNewton, TimeShardedNewton, block_bounds
logT = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T, nx, nu, damp = 1 << logT, 12, 4, 0.9999
dev = torch.device("cuda")
f64 = torch.float64
g = torch.Generator(device=dev).manual_seed(20028)
band = torch.zeros(nx, nx, dtype=f64, device=dev)
for i in range(4):
    for j in (i, i + 1):
        if j < 4:
            band[3 * i:3 * i + 3, 3 * j:3 * j + 3] = 1.0
F = torch.randn(T, nx, nx, generator=g, device=dev, dtype=f64) * (0.2 ** 0.5) * band
A = (damp * (torch.eye(nx, dtype=f64, device=dev) + 0.01 * F)).cpu().numpy()
del F
Bm = (torch.randn(T, nx, nu, generator=g, device=dev, dtype=f64) * (0.1 ** 0.5)).cpu().numpy()
qd = torch.empty(nx, dtype=f64, device=dev).uniform_(0.1, 10.0, generator=g).cpu().numpy()
x0 = torch.randn(nx, generator=g, device=dev, dtype=f64).cpu().numpy()
cost = P.QuadraticCost(np.diag(qd), 0.1 * np.eye(nu), 10 * np.diag(qd))
box = P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-4)
st = SolveSettings(method=N.METHOD_BARRIER, max_iters=50, mu0=0.1, zeta=0.2, mu_tol=1e-4,
                   round_cap=opts.rounds())
for world in (1, 2, 4, 8):
    blocks, U = [], []
    for r in range(world):
        t0, m = block_bounds(T, world, r)
        dyn = P.TimeVaryingLinearDynamics(A[t0:t0 + m], Bm[t0:t0 + m])
        blocks.append(BlockNewton(dyn, cost, box, 1, st, r, world, t0))
        U.append(np.zeros((1, m, nu)))
    drv = TimeShardedNewton(blocks, emulate=True)
    drv.set_initial_state(x0[None])
    X = drv.rollout(U)
    drv.solve(X, U)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    drv.solve(X, U)
    b.record()
    torch.cuda.synchronize()
    s = blocks[0].solver
    n = int(s.read("round")[0])
    its = int(s.rounds("round_iters")[:n, 0].sum())
    tot = a.elapsed_time(b)
    print({"world": world, "total_ms": round(tot, 2), "per_rank_ms": round(tot / world, 2),
           "iters": its, "per_rank_ms_per_iter": round(tot / world / its, 3),
           "cost": float(s.read("cur_cost")[0])}, flush=True)
    del blocks, drv, X
    torch.cuda.empty_cache()
