"""c5 at M=2048: GPU pipeline timing on a slice of blocks, and one block against
the reference's block_svd (keep 64). Not collected by pytest (long)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import compare
cfg = configs.CONFIGS["c5"]
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t = time.time()
a = cfg.generate(nb * 16384)
print("generated", a.nnz(), time.time() - t, flush=True)
dm = rk.DeviceMatrix(a)
for it in range(2):
    out, tm = rk.ranky.dev_full_svd(dm, nb, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    rk.ranky.dev_outputs_free(out)
    print("device", tm.as_dict(), flush=True)
if len(sys.argv) > 2:
    from oracle import Oracle
    ref = Oracle("reference")
    p = rk.partition_columns(a.cols(), nb)
    rep, report = rk.repair(a, p, cfg.method, cfg.seed)
    b = rk.block_view(rep, p, 0)
    t = time.time()
    g = rk.block_svd(b, 64)
    print("gpu block", time.time() - t, flush=True)
    r, c, v = b.coo()
    t = time.time()
    o = ref.block_svd((b.rows(), b.cols(), r, c, v), 64)
    print("ref block", time.time() - t, flush=True)
    compare(g, o.sigma, o.u, "c5 block 0")
    print("block 0 sigma rel", float(np.max(np.abs(g.sigma - o.sigma) / o.sigma)), flush=True)
