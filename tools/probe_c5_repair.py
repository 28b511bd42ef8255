"""Device repair of the full-size c5 matrix (NeighborRandomChecker): time of
rk.repair (H2D, the ordered replay, D2H) and of the device-resident pipeline's
repair stage. python tools/probe_c5_repair.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402

cfg = configs.CONFIGS["c5"]
t0 = time.perf_counter()
a = cfg.generate()
print(f"generated {a.nnz()} nnz in {time.perf_counter() - t0:.1f} s", flush=True)
p = rk.partition_columns(a.cols(), cfg.blocks)
for it in range(2):
    t0 = time.perf_counter()
    rep, report = rk.repair(a, p, cfg.method, cfg.seed)
    print(f"rk.repair: {time.perf_counter() - t0:.2f} s, {len(report.added_edges)} edges, "
          f"{report.fallback_count} fallbacks, first edges {report.edges_array()[:2].tolist()}", flush=True)
