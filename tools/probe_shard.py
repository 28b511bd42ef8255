"""Per-rank device time of the sharded pipeline (weak scaling: c2 tiled ws times),
estimated on one GPU: rank 0's rk_dev_shard_factor, the gathered factors stood in
by copies of its own (the NCCL all-gather of ws x 512 KiB is not timed), and
rk_dev_shard_finish. python tools/probe_shard.py [ws ...]"""
import ctypes as C
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs, ranky as R, shard as SH  # noqa: E402

L = R.lib()
ROUTE = os.environ.get("RK_SHARD_ROUTE", "gram")  # gram | tsqr
ctx = rk.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
for ws in [int(x) for x in sys.argv[1:]] or [1, 8]:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    cfg = dataclasses.replace(configs.CONFIGS["c2"], cols=262144 * ws, blocks=64 * ws)
    a = bench.weak_matrix(configs.CONFIGS["c2"], ws, R) if ws > 1 else cfg.generate()
    dm = rk.DeviceMatrix(a, ctx)
    M = cfg.rows
    sp = SH.plan(M, cfg.cols, cfg.blocks, cfg.keep, ws, 0)
    roots = torch.empty((ws, M, M), dtype=torch.float64, device="cuda")
    mine = torch.empty((M, M), dtype=torch.float64, device="cuda")
    ts = []
    for it in range(6):
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        shard = C.c_void_p()
        t = R.Timing()
        fac = L.rk_dev_shard_factor_gram if ROUTE == "gram" else L.rk_dev_shard_factor
        R._check(fac(ctx.handle, dm.handle, cfg.blocks, R._method(cfg.method), cfg.keep, cfg.seed,
                     sp.leaf_lo, sp.leaf_hi, C.c_void_p(mine.data_ptr()), C.byref(shard), C.byref(t)))
        e1.record(stream)
        roots.copy_(mine.unsqueeze(0).expand(ws, M, M))
        out = C.POINTER(R.DevOutputs)()
        t2 = R.Timing()
        fin = L.rk_dev_shard_finish_gram if ROUTE == "gram" else L.rk_dev_shard_finish
        R._check(fin(ctx.handle, shard, C.c_void_p(roots.data_ptr()), ws, R.WANT_V, cfg.top_k,
                     sp.col_lo, sp.col_hi, C.byref(out), C.byref(t2)))
        e2.record(stream)
        torch.cuda.synchronize()
        R.dev_outputs_free(out)
        L.rk_dev_shard_destroy(shard)
        if it >= 2:
            ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2), t.blocks_ms, t.merge_ms, t.repair_ms, t2.merge_ms))
            det = (t.qr_ms, t.jacobi_ms, t.jacobi_sweeps_max, t.kernel_launches)
    f = [sum(x[i] for x in ts) / len(ts) for i in range(6)]
    print(f"[{ROUTE}] ws={ws}: factor {f[0]:.2f} ms (repair {f[4]:.2f}, blocks {f[2]:.2f}, subtree merge {f[3]:.2f}), "
          f"finish {f[1]:.2f} ms (merge {f[5]:.2f}); total {f[0] + f[1]:.2f} ms; nnz/s per rank x ws = "
          f"{a.nnz() / ((f[0] + f[1]) / 1e3):.3e}; qr/gram {det[0]:.2f} jacobi {det[1]:.2f} sweeps {det[2]} "
          f"launches {det[3]}")
    dm.close()
