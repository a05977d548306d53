"""Per-rank headline workload of an N-GPU strong-scaling run, timed on one
GPU (rank 0's share: 65,536 / N problems), for several scan plans."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver

out = {}
for world in (1, 2, 4, 8):
    b_local = bench.B_TOTAL // world
    bp, bc = bench.half_sizes(b_local)
    halves = {}
    for system, n in (("pendulum", bp), ("cartpole", bc)):
        inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
        probe = LqrSolver(n, bench.T, nx, nu)
        alpha = bench.lm_alpha_device(torch, probe, inputs, n)
        halves[system] = (inputs, alpha, n, nx, nu)
    for plan in ((0, 0), (bench.T, 0), (64, 4), (32, 8)):
        sols = {k: LqrSolver(h[2], bench.T, h[3], h[4], chunk0=plan[0], chunk=plan[1])
                for k, h in halves.items()}
        side = [torch.cuda.Stream() for _ in sols]
        main = torch.cuda.current_stream()

        def step():
            for st in side:
                st.wait_stream(main)
            for (k, sol), st in zip(sols.items(), side):
                with torch.cuda.stream(st):
                    sol.solve(*halves[k][0], halves[k][1], stream=st)
            for st in side:
                main.wait_stream(st)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            step()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        out[f"N{world}_plan{plan}"] = {"ms": round(ms, 4), "plan": sols["cartpole"].plan(),
                                      "solves_per_s_all_ranks": round(bench.B_TOTAL / (ms * 1e-3))}
        del sols
    del halves
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
