"""e2e (host buffers) throughput vs sub-batch count and stream count."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import HostLqrSolver, LqrSolver
T = bench.T
halves = {}
for system in ("pendulum", "cartpole"):
    inputs, nx, nu = bench.build_inputs(P, torch, system, 32768, 0)
    alpha = bench.lm_alpha_device(torch, LqrSolver(32768, T, nx, nu), inputs, 32768)
    halves[system] = (inputs, alpha, 32768, nx, nu)
res = {}
for nsub in (4, 8, 16):
    subs = []
    for k, (inputs, alpha, n, nx, nu) in halves.items():
        st_ = n // nsub
        for i in range(nsub):
            sl = slice(i * st_, n if i == nsub - 1 else (i + 1) * st_)
            m = sl.stop - sl.start
            h_in = [t[:, :, sl].contiguous().cpu().pin_memory() for t in inputs]
            h_al = alpha[sl].contiguous().cpu().pin_memory()
            hs = HostLqrSolver(m, T, nx, nu)
            subs.append((hs, h_in, h_al, hs.outputs()))
    for ns in (2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        def step():
            main = torch.cuda.current_stream()
            for s in streams:
                s.wait_stream(main)
            for k, (hs, h_in, h_al, h_out) in enumerate(subs):
                hs.solve(*h_in, h_al, h_out, stream=streams[k % ns])
            for s in streams:
                main.wait_stream(s)
        step(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            step()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 4
        res[f"nsub{nsub}_streams{ns}"] = round(65536 / (ms * 1e-3) / 1e6, 4)
        print(nsub, ns, ms, flush=True)
    del subs
print(json.dumps(res))
