import faulthandler, sys, os, time
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2409_20027_b200 as P
from paper_2409_20027_b200 import usermodel
from user_models import user_pendulum, user_tvlinear
t0 = time.time()
dyn = user_pendulum(8)
print("lib", dyn.library(), time.time() - t0, flush=True)
print("load", usermodel.load_model(dyn.library()), time.time() - t0, flush=True)
spec = dyn._device_spec(); print("spec", spec, flush=True)
tr = P.rollout(dyn, np.array([0.1, 0.0]), np.zeros((8, 1)))
print("rollout ok", tr.states[-1], time.time() - t0, flush=True)
ref = P.rollout(P.PendulumDynamics(8, P.PendulumParams(damping=0.1, dt=0.05)), np.array([0.1, 0.0]), np.zeros((8, 1)))
print("builtin", ref.states[-1], flush=True)
