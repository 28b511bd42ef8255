import time, torch
n = 537 * 2**20 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("D2H GB/s", n * 8 / dt / 1e9)
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("H2D GB/s", n * 8 / dt / 1e9)
# two streams, two halves
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2:].copy_(d[n // 2:], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("D2H 2 streams GB/s", n * 8 / dt / 1e9)
