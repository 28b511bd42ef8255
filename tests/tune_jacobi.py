"""Tuning probe (not collected by pytest): block-Jacobi time on c2 for several
(RK_JACOBI_GMAX, RK_JACOBI_Q) settings, read back from the pipeline timing."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
cfg = configs.CONFIGS["c2"]
a = cfg.generate()
dm = rk.DeviceMatrix(a)
for gmax, q in [(16, "16"), (32, "8"), (8, "32")]:
    os.environ["RK_JACOBI_GMAX"] = str(gmax)
    os.environ["RK_JACOBI_Q"] = q
    ts = []
    for _ in range(4):
        out, t = rk.ranky.dev_full_svd(dm, cfg.blocks, cfg.method, 0, cfg.seed, True, 0)
        rk.ranky.dev_outputs_free(out)
        ts.append((t.jacobi_ms, t.merge_ms, t.total_ms, t.jacobi_sweeps_max))
    j = statistics.median(x[0] for x in ts[1:]); m = statistics.median(x[1] for x in ts[1:])
    print(f"gmax={gmax:2d} Q={q:>2}: block jacobi {j:7.3f} ms  merge {m:7.3f} ms  total {ts[-1][2]:7.3f}  sweeps {ts[-1][3]}", flush=True)
