"""The headline step (both config-3 halves concurrently on two streams) with
the pendulum half on different scan plans; per-GPU batch n per half."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2409_20027_b200 as P
from paper_2409_20027_b200.passes import LqrSolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pin, pnx, pnu = bench.build_inputs(P, torch, "pendulum", n, 0)
cin, cnx, cnu = bench.build_inputs(P, torch, "cartpole", n, 0)
alpha = torch.full((n,), 64.0, dtype=torch.float64, device="cuda")
cs = LqrSolver(n, bench.T, cnx, cnu)
out = {}
for name, c0 in (("sweep", bench.T), ("k128", 128), ("k64", 64), ("k32", 32)):
    ps = LqrSolver(n, bench.T, pnx, pnu, chunk0=c0, chunk=8 if c0 < bench.T else 0)
    st = [torch.cuda.Stream(), torch.cuda.Stream()]
    main = torch.cuda.current_stream()
    def step():
        for s in st: s.wait_stream(main)
        with torch.cuda.stream(st[0]): ps.solve(*pin, alpha, stream=st[0])
        with torch.cuda.stream(st[1]): cs.solve(*cin, alpha, stream=st[1])
        for s in st: main.wait_stream(s)
    for _ in range(3): step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): step()
    b.record(); torch.cuda.synchronize()
    out[name] = round(a.elapsed_time(b) / 20, 4)
    del ps
print(n, json.dumps(out))
