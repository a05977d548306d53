"""Headline step (config 3 LQR-scan solves, 65,536 problems) under different
launch orders / stream priorities of its two halves: ms per step."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver

halves = {}
for system, n in (("pendulum", 32768), ("cartpole", 32768)):
    inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
    solver = LqrSolver(n, bench.T, nx, nu, dtype=torch.float64)
    alpha = bench.lm_alpha_device(torch, solver, inputs, n)
    halves[system] = (solver, inputs, alpha)
torch.cuda.synchronize()
stream = torch.cuda.current_stream()


def variant(order, prio):
    side = [torch.cuda.Stream(priority=p) for p in prio]
    def step():
        for st in side:
            st.wait_stream(stream)
        for k, st in zip(order, side):
            solver, inputs, alpha = halves[k]
            with torch.cuda.stream(st):
                solver.solve(*inputs, alpha, stream=st)
        for st in side:
            stream.wait_stream(st)
    return step


def seq():
    for k in ("cartpole", "pendulum"):
        solver, inputs, alpha = halves[k]
        solver.solve(*inputs, alpha)


variants = {
    "pend_first": variant(("pendulum", "cartpole"), (0, 0)),
    "cart_first": variant(("cartpole", "pendulum"), (0, 0)),
    "cart_first_prio_cart": variant(("cartpole", "pendulum"), (-1, 0)),
    "pend_first_prio_cart": variant(("pendulum", "cartpole"), (0, -1)),
    "pend_first_prio_pend": variant(("pendulum", "cartpole"), (-1, 0)),
    "sequential": seq,
}
for rep in range(2):
    for name, fn in variants.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(20):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        print(json.dumps({"variant": name, "ms": round(a.elapsed_time(b) / 20, 4)}), flush=True)
