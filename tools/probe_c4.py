"""c4 (1024 x 16.8M) device pipeline timing and memory (development tool)."""
import sys, os, time
sys.path.insert(0, "/root/repo")
import torch
print("mem_get_info", [x / 2**30 for x in torch.cuda.mem_get_info()], flush=True)
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
cfg = configs.CONFIGS["c4"]
a = cfg.generate()
dm = rk.DeviceMatrix(a)
t0 = time.time()
try:
    out, t = rk.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    print("ok", time.time() - t0, t.as_dict(), flush=True)
except Exception as e:
    print("fail", e, flush=True)
print("mem_get_info", [x / 2**30 for x in torch.cuda.mem_get_info()], flush=True)
