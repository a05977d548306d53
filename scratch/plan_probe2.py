"""Two-stream config-3 step (both halves concurrently, as bench.py times it)
for scan-plan combinations at the per-GPU batch of N = 1, 2, 4, 8."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
T = bench.T
cands = [(T, 0), (128, 8), (64, 8), (64, 16), (32, 16), (32, 8), (16, 4), (16, 16)]
for n in (4096, 8192, 16384, 32768):
    halves = {}
    for system in ("pendulum", "cartpole"):
        inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
        alpha = bench.lm_alpha_device(torch, LqrSolver(n, T, nx, nu), inputs, n)
        halves[system] = (inputs, alpha, nx, nu)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    res = {}
    for pp, cp in itertools.product(cands, cands):
        solvers = [LqrSolver(n, T, halves[s][2], halves[s][3], chunk0=c[0], chunk=c[1])
                   for s, c in (("pendulum", pp), ("cartpole", cp))]
        def step():
            main = torch.cuda.current_stream()
            for st in streams:
                st.wait_stream(main)
            for (s, st, key) in zip(solvers, streams, ("pendulum", "cartpole")):
                inputs, alpha, _, _ = halves[key]
                s.solve(*inputs, alpha, stream=st)
            for st in streams:
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
        res[f"{pp[0]}/{pp[1]}|{cp[0]}/{cp[1]}"] = round(a.elapsed_time(b) / 10, 4)
        del solvers
    best = sorted(res.items(), key=lambda kv: kv[1])[:5]
    print(json.dumps({"n_per_half": n, "sweep|sweep": res[f"{T}/0|{T}/0"], "best5": best}),
          flush=True)
    del halves
    torch.cuda.empty_cache()
