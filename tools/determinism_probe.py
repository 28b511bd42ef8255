"""Determinism of the device pipeline and of the sharded protocol (c3 by default):
the same call twice must give the same bits, and every rank's Gram-route decision
must agree. Ranks run one after another in this process (tests/test_gpu_shard.py's
protocol).

    python tools/determinism_probe.py [c3]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402
from paper_2009_09767_b200 import ranky as R  # noqa: E402
from test_gpu_shard import run_sharded  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = configs.CONFIGS[name]
dm = rk.DeviceMatrix(cfg.generate())
for eig in ("1", "0"):
    os.environ["RK_EIG_MERGE"] = eig
    R.reload_tuning()
    runs = []
    for i in range(3):
        out, t = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
        sig, u, v = R.dev_outputs_tensors(out)
        runs.append((sig.cpu().numpy(), u.cpu().numpy(), v[:4096].cpu().numpy()))
        R.dev_outputs_free(out)
    same = [all(np.array_equal(a, b) for a, b in zip(runs[0], r)) for r in runs[1:]]
    print(f"eig={eig} dev_full_svd repeat bitwise: {same}", flush=True)
    for world in (2, 4):
        res = [run_sharded(dm, cfg, world, route="gram") for _ in range(2)]
        (o1, g1), (o2, g2) = res
        eq = all(np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2]) for x, y in zip(o1, o2))
        ranks_eq = all(np.array_equal(o1[0][1], x[1]) and np.array_equal(o1[0][2], x[2]) for x in o1)
        print(f"eig={eig} world={world}: gram route {g1}/{g2}, repeat bitwise {eq}, ranks agree {ranks_eq}",
              flush=True)
