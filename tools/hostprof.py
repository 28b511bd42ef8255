"""Host/device segment times of one device pipeline call (RK_HOSTPROF=1).

    RK_HOSTPROF=1 python tools/hostprof.py c3 [calls]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402
from paper_2009_09767_b200.ranky import dev_full_svd, dev_outputs_free  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dm = rk.DeviceMatrix(cfg.generate())
for i in range(calls):
    out, t = dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    print(f"call {i}: {t.as_dict()}", flush=True)
    dev_outputs_free(out)
