import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RK_JACOBI_CHECK"] = "1"
import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
cfg = configs.CONFIGS["c2"]
a = cfg.generate()
dm = rk.DeviceMatrix(a)
out, t = rk.ranky.dev_full_svd(dm, cfg.blocks, cfg.method, 0, cfg.seed, True, 0)
print(t.as_dict())
