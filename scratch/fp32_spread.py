"""fp32 reproducibility of the test_gpu_fp32 cart-pole instance: the device
fp32 barrier solve from u0 nudged by one float32 ulp (random signs), its
rounds and its gap to the fp64 oracle."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2409_20027_b200 as P
from oracle import pintoc_oracle as O
from test_gpu_fp32 import _cartpole, _gap, _f32
prob, (od, oc, ob) = _cartpole(P, 48, state_box=False)
kw = dict(inner_tol=1e-5, max_iters=200)
cases = {"T48_dth0.2": np.array([0.1, math.pi - 0.2, 0.0, 0.1]),
         "T48_dth0.1": np.array([0.1, math.pi - 0.1, 0.0, 0.05]),
         "T48_dth0.05": np.array([0.0, math.pi - 0.05, 0.0, 0.0]),
         "T48_dth0.15": np.array([0.05, math.pi - 0.15, 0.0, 0.0])}
for name, x0 in cases.items():
  rng = np.random.default_rng(11)
  u0 = 0.5 * rng.standard_normal((48, 1))
  ref = O.barrier_solve(od, oc, ob, O.rollout(od, _f32(x0), _f32(u0)), _f32(u0), **kw)
  print(name, "oracle", [q.iterations for q in ref.newton], "max|u|", float(np.abs(ref.us).max()))
  r2 = np.random.default_rng(5)
  for k in range(6):
    u32 = np.asarray(u0, np.float32)
    if k:
        sgn = r2.choice([-1, 1], size=u32.shape)
        u32 = np.where(sgn > 0, np.nextafter(u32, np.float32(np.inf)), np.nextafter(u32, np.float32(-np.inf)))
    init = P.rollout(prob.dynamics, x0, u32.astype(np.float64))
    traj, rep = P.barrier_solve(prob, init, P.BarrierOptions(newton=P.NewtonOptions(**kw)), dtype=torch.float32)
    print(" ", k, [r.newton.iterations for r in rep.rounds], f"gap {_gap(traj.controls, ref.us):.2e}", flush=True)
