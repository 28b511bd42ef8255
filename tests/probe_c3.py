"""Debug probe (not collected by pytest): c3 block / pipeline timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
cfg = configs.CONFIGS["c3"]
what = sys.argv[1]
if what == "block":
    a = cfg.generate()
    p = rk.partition_columns(a.cols(), cfg.blocks)
    for d in (0, 56, 133):
        b = rk.block_view(a, p, d)
        t = time.time()
        s = rk.block_svd(b, 512)
        print("block", d, b.nnz(), time.time() - t, s.sigma[:3], s.sigma[-3:], flush=True)
elif what == "pipe":
    n = int(sys.argv[2])
    a = cfg.generate(8192 * n)
    t = time.time()
    res = rk.run_pipeline(a, n, cfg.method, 0, cfg.seed, 1, want_v=False)
    print("pipe", n, time.time() - t, res.timing, flush=True)
