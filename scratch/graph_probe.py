import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import _native as N
from paper_2409_20027_b200._device import SolveSettings
from paper_2409_20027_b200.sharded import BlockNewton, TimeShardedNewton, block_bounds
T, nx, nu = 1 << 18, 12, 4
rng = np.random.default_rng(1)
A = np.eye(nx)[None] * 0.9999 + 0.004 * rng.standard_normal((T, nx, nx))
B = 0.3 * rng.standard_normal((T, nx, nu))
cost = P.QuadraticCost(np.eye(nx), 0.1 * np.eye(nu), 10 * np.eye(nx))
box = P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
st = SolveSettings(method=N.METHOD_BARRIER, max_iters=50, round_cap=5)
dyn = P.TimeVaryingLinearDynamics(A, B)
blk = BlockNewton(dyn, cost, box, 1, st, 0, 1, 0)
drv = TimeShardedNewton([blk], emulate=True)
drv.set_initial_state(rng.standard_normal(nx)[None])
U = [np.zeros((1, T, nu))]
X = drv.rollout(U)
for k, bl in enumerate(drv.blocks):
    bl.solver.load(X[k], U[k])
drv.iteration(); torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
a, b = ev(), ev(); a.record()
for _ in range(3): drv.iteration()
b.record(); torch.cuda.synchronize(); print("eager ms/it", a.elapsed_time(b) / 3)
g = drv._capture(); print("graph", g is not None)
torch.cuda.synchronize()
a, b = ev(), ev(); a.record()
for _ in range(3): g.replay()
b.record(); torch.cuda.synchronize(); print("replay ms/it", a.elapsed_time(b) / 3)
a, b = ev(), ev(); a.record()
for _ in range(3): drv.iteration()
b.record(); torch.cuda.synchronize(); print("eager again ms/it", a.elapsed_time(b) / 3)
