import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs, ranky as R
cfg = configs.CONFIGS["c2"]
a = cfg.generate()
ctx = rk.Context(0)
pinned = torch.empty(a.nnz() * R.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
host_e = pinned.numpy().view(R.ENTRY_DTYPE)
host_e[:] = a.entries()
ha = R.SparseMatrix._trusted(a.rows(), a.cols(), host_e)
import ctypes as C
L = R.lib()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = R._Pipeline()
    v = ha._view()
    st = L.rk_run_pipeline(ctx.handle, C.byref(v), cfg.blocks, R._method(cfg.method), 0, cfg.seed, 1, R.WANT_V, 0, C.byref(out))
    t1 = time.perf_counter()
    L.rk_pipeline_result_free(C.byref(out))
    t2 = time.perf_counter()
    res = rk.run_pipeline(ha, cfg.blocks, cfg.method, 0, cfg.seed, 1, want_v=True, want_repaired=False, want_records=False, ctx=ctx)
    t3 = time.perf_counter()
    print(f"raw call {1e3*(t1-t0):.2f} ms (device total {out.timing.total_ms:.2f}), free {1e3*(t2-t1):.2f}, wrapper call {1e3*(t3-t2):.2f} (device {res.timing['total_ms']:.2f})", flush=True)
