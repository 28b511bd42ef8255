"""Pure-write HBM bandwidth (torch fill / cudaMemset) next to the copy rate in MEASURED_PEAKS.json:
the roof of the V recovery, which writes 8 N r bytes and reads almost nothing."""
import torch
for gib in (4, 16, 64):
    n = gib * 2**30 // 8
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        x.zero_()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); x.zero_(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"fill {gib} GiB: {best:.3f} ms = {gib * 2**30 / best / 1e6:.0f} GB/s", flush=True)
    y = torch.empty(n // 2, dtype=torch.float64, device="cuda"); z = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); z.copy_(y); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"copy {gib // 2} GiB -> {gib // 2} GiB: {best:.3f} ms = {gib * 2**30 / best / 1e6:.0f} GB/s (read + write)", flush=True)
    del x, y, z
    torch.cuda.empty_cache()
