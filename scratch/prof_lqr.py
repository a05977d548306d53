"""Profile driver: one batch-1 LQR-scan solve (config-1 generator), args nx logT [reps] [chunk0 chunk]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.pintoc_oracle import random_lqr_expansion
from paper_2409_20027_b200.passes import LqrSolver
nx, logT = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c0, c1 = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 0)
nu, Tn = nx // 2, 1 << logT
e = random_lqr_expansion(np.random.default_rng([1, nx, logT]), Tn, nx, nu)
soa = lambda a, c: torch.as_tensor(a.reshape(a.shape[0], c).T.copy()).unsqueeze(-1).cuda()
ins = [soa(e.P, nx * nx), soa(e.R, nu * nu), soa(e.M, nx * nu), soa(e.d, nu), soa(e.Fx, nx * nx),
       soa(e.Fu, nx * nu), soa(e.PT[None], nx * nx)]
alpha = torch.zeros(1, dtype=torch.float64, device="cuda")
s = LqrSolver(1, Tn, nx, nu, chunk0=c0, chunk=c1)
print("plan", s.plan())
for _ in range(2):
    s.solve(*ins, alpha)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    s.solve(*ins, alpha)
b.record()
torch.cuda.synchronize()
print("ms", a.elapsed_time(b) / reps, "flags", int(s.flags[0]))
