"""Tuning probe (not collected by pytest): c2 stage times for Jacobi variants."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
cfg = configs.CONFIGS["c2"]
a = cfg.generate()
dm = rk.DeviceMatrix(a)
variants = [dict(), dict(RK_JACOBI_UNROLL="0")]
for env in variants:
    for k in ("RK_JACOBI_DIRECT", "RK_JACOBI_GMAX", "RK_JACOBI_Q", "RK_JACOBI_CHECK", "RK_JACOBI_WARP", "RK_JACOBI_SINGLE_G", "RK_JACOBI_CLUSTER", "RK_JACOBI_UNROLL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ts = []
    for _ in range(4):
        out, t = rk.ranky.dev_full_svd(dm, cfg.blocks, cfg.method, 0, cfg.seed, True, 0)
        rk.ranky.dev_outputs_free(out)
        ts.append((t.jacobi_ms, t.merge_ms, t.total_ms, t.jacobi_sweeps_max, t.jacobi_sweeps_sum))
    med = [statistics.median(x[i] for x in ts[1:]) for i in range(3)]
    print(f"{str(env):32s}: block jacobi {med[0]:7.3f} ms  merge {med[1]:7.3f} ms  total {med[2]:7.3f}  sweeps max {ts[-1][3]} sum {ts[-1][4]}", flush=True)
