import torch, time
n = 1 << 27   # 1 GiB of fp64
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, src, dst in (("h2d", h, d), ("d2h", d, h)):
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): dst.copy_(src, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    print(name, round(5 * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9, 2), "GB/s")
# both directions at once on two streams
h2 = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("duplex", round(5 * 8 * n / dt / 1e9, 2), "GB/s each way")
