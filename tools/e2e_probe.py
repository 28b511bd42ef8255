"""Where the e2e time of the host-buffer C-ABI call goes (c3 by default):
pinned D2H bandwidth of a V-sized buffer (torch), then rk_run_pipeline with
RK_HOSTPROF=1 (library segments) and the Python wrapper's share.

    RK_HOSTPROF=1 python tools/e2e_probe.py [c3]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402
from paper_2009_09767_b200 import ranky as R  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = cfg.cols * cfg.rows
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"torch pinned D2H {8 * n / 2**30:.1f} GiB: {dt * 1e3:.1f} ms = {8 * n / dt / 1e9:.1f} GB/s", flush=True)
del d, h
a = cfg.generate()
pinned = torch.empty(a.nnz() * R.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
he = pinned.numpy().view(R.ENTRY_DTYPE)
he[:] = a.entries()
ha = R.SparseMatrix._trusted(a.rows(), a.cols(), he)
ctx = rk.Context(0)
for i in range(3):
    t0 = time.perf_counter()
    res = rk.run_pipeline(ha, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True, top_k=cfg.top_k, ctx=ctx)
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt * 1e3:.1f} ms (device total {res.timing['total_ms']:.1f} ms)", flush=True)
    del res
