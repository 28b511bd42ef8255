import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
mode = sys.argv[1]
os.environ["RK_JACOBI_CHECK"] = mode
rng = np.random.default_rng(0)
for n in (64, 256):
    a = rng.standard_normal((n, n))
    try:
        s = rk.dense_svd(a)
        print(mode, "dense", n, np.abs(s.sigma - np.linalg.svd(a, compute_uv=False)).max() / s.sigma[0], flush=True)
    except Exception as e:
        print(mode, "dense", n, "FAIL", e, flush=True)
for name in ("c1", "c2"):
    cfg = configs.CONFIGS[name]
    a = cfg.generate()
    try:
        res = rk.run_pipeline(a, cfg.blocks, cfg.method, 0, cfg.seed, 1)
        print(mode, name, res.timing["jacobi_sweeps_max"], res.timing["jacobi_sweeps_sum"], res.timing["jacobi_ms"], flush=True)
    except Exception as e:
        print(mode, name, "FAIL", e, flush=True)
