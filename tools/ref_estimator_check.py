"""Validate bench.py's stage-sampled reference estimator against one full reference
run on the same host (run on the GPU box: 16 cores):

    python tools/ref_estimator_check.py c3
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = configs.CONFIGS[name]
a = cfg.generate()
cores = os.cpu_count() or 1
est = bench.ReferenceEstimator(cfg, a, cores)
t0 = time.perf_counter()
first, parts = est.calibrate()
steps = [est.step()[0] for _ in range(3)]
t_est = time.perf_counter() - t0
r, c, v = a.coo()
orc = Oracle("reference")
t0 = time.perf_counter()
res = orc.full_svd((a.rows(), a.cols(), r, c, v), cfg.blocks, cfg.method, cfg.keep, cfg.seed, cores, cfg.top_k)
wall = time.perf_counter() - t0
full = res.times[1] + res.times[2]
print(json.dumps({"config": name, "cores": cores, "cpu_model": bench.cpu_model(),
                  "estimate_s": [first] + steps, "estimate_parts_first": parts, "calibration": est.calib,
                  "estimator_wall_s": t_est, "full_run_pipeline_s": res.times[1], "full_recover_s": res.times[2],
                  "full_total_s": full, "full_wall_incl_marshalling_s": wall}, default=float))
