"""Config 2 (cart-pole ADMM, T=500) per-iteration timing probe."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2409_20027_b200 as P
outer = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ex = sys.argv[2] if len(sys.argv) > 2 else "auto"
probs = bench.models_pkg(P)
cart = probs["cartpole"]
T2 = 500
cart = P.ControlProblem(P.CartPoleDynamics(T2, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                                pole_length=0.5, dt=0.02)),
                        cart.cost, cart.constraints)
rng = np.random.default_rng(20027)
rng.standard_normal((100, 1))
u2 = np.clip(1.0 * rng.standard_normal((T2, 1)), -9.0, 9.0)
init2 = P.rollout(cart.dynamics, np.zeros(4), u2)
o2 = P.AdmmOptions(rho=1.0, max_outer=outer, newton=P.NewtonOptions(executor=ex))
P.admm_solve(cart, init2, o2)
torch.cuda.synchronize()
t = time.perf_counter()
_, rep2 = P.admm_solve(cart, init2, o2)
torch.cuda.synchronize()
g2 = time.perf_counter() - t
print({"executor": ex, "s": round(g2, 4), "iters": rep2.inner_iterations,
       "ms_per_iter": round(1e3 * g2 / rep2.inner_iterations, 4)})
