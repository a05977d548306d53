"""Strong-scaling shares of the headline (65,536 / N problems, both models
concurrently, T = 256) on one GPU: the automatic plan vs the single sweep
on the register path vs the single sweep on TMA-fed rings (PTC_BULK=1;
one-warp CTAs below 16,384 problems).  ms per step."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver

for world in (1, 2, 4, 8, 16):
    b_local = bench.B_TOTAL // world
    bp, bc = bench.half_sizes(b_local)
    halves = {}
    for system, n in (("pendulum", bp), ("cartpole", bc)):
        inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
        probe = LqrSolver(n, bench.T, nx, nu)
        alpha = bench.lm_alpha_device(torch, probe, inputs, n)
        halves[system] = (inputs, alpha, n, nx, nu)
    res = {}
    ref = None
    for name, plan, bulk in (("auto", (0, 0), "0"), ("sweep_regs", (bench.T, 0), "0"),
                             ("sweep_ring", (bench.T, 0), "1")):
        os.environ["PTC_BULK"] = bulk
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
        for _ in range(20):
            step()
        b.record()
        torch.cuda.synchronize()
        out = torch.cat([s.du.flatten() for s in sols.values()])
        if ref is None:
            ref = out.clone()
        res[name] = {"ms": round(a.elapsed_time(b) / 20, 4),
                     "max_gap_vs_auto": float((out - ref).abs().max())}
    print(json.dumps({"N": world, "per_rank": b_local, **res}), flush=True)
