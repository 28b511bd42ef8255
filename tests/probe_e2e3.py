import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs, ranky as R
cfg = configs.CONFIGS["c2"]
a = cfg.generate()
mode = sys.argv[1]
ctx = rk.Context(0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
if "dev" in mode:
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    dm = rk.DeviceMatrix(a, ctx)
    for _ in range(13):
        out, t = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
        R.dev_outputs_free(out)
        flush.zero_()
    torch.cuda.synchronize()
pinned = torch.empty(a.nnz() * R.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
host_e = pinned.numpy().view(R.ENTRY_DTYPE)
host_e[:] = a.entries()
ha = R.SparseMatrix._trusted(a.rows(), a.cols(), host_e)
ctx_e = rk.Context(0)
for _ in range(3):
    rk.run_pipeline(ha, cfg.blocks, cfg.method, 0, cfg.seed, 1, want_v=True, want_repaired=False, want_records=False, ctx=ctx_e)
ts = []
for it in range(20):
    if "flush" in mode:
        flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = rk.run_pipeline(ha, cfg.blocks, cfg.method, 0, cfg.seed, 1, want_v=True, want_repaired=False, want_records=False, ctx=ctx_e)
    ts.append(round(1e3 * (time.perf_counter() - t0), 1))
print(mode, ts, flush=True)
