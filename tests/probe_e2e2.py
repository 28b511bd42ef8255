import os, sys, time, gc
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
for mode in ("gc", "nogc"):
    if mode == "nogc":
        gc.disable()
    ts = []
    res = None
    for it in range(20):
        t0 = time.perf_counter()
        res = rk.run_pipeline(ha, cfg.blocks, cfg.method, 0, cfg.seed, 1, want_v=True, want_repaired=False, want_records=False, ctx=ctx)
        ts.append(round(1e3 * (time.perf_counter() - t0), 1))
    print(mode, ts, flush=True)
