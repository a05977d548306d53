import faulthandler, sys, os, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import usermodel
from user_models import user_pendulum, user_tvlinear
t0 = time.time()
g = np.load("tests/golden/barrier_tvlinear.npz")
dyn = user_tvlinear(g["A"], g["B"], g["c"])
print("lib", dyn.library(), time.time() - t0, flush=True)
spec = dyn._device_spec(); print("spec", spec["model"], time.time() - t0, flush=True)
tr = P.rollout(dyn, g["x0"], g["u0"])
print("rollout ok", tr.states[-1], time.time() - t0, flush=True)
ref = P.rollout(P.TimeVaryingLinearDynamics(g["A"], g["B"], g["c"]), g["x0"], g["u0"])
print("builtin", ref.states[-1], flush=True)
