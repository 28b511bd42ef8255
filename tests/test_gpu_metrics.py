"""GPU reconstruction residual (rk_dev_residual) against numpy on the dense
repaired matrix -- the reference's reconstruction metric (proj/tests/
test_support.hpp:57-70; svd_test.cpp:302-339 requires <= 1e-10 relative for a
full decomposition)."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200 import ranky as R

pytestmark = pytest.mark.gpu


def dense_residual(rep, u, sigma, v):
    a = rep.to_dense()
    return float(np.linalg.norm(a - (u * sigma) @ v.T)), float(np.linalg.norm(a))


@pytest.mark.parametrize("case", ["c1", "c2slice", "c5shape"])
def test_device_residual_matches_dense(case):
    if case == "c1":
        cfg = configs.CONFIGS["c1"]
        a, blocks, method, keep, seed, top_k = cfg.generate(), cfg.blocks, cfg.method, 0, cfg.seed, 0
    elif case == "c2slice":
        cfg = configs.CONFIGS["c2"]
        a, blocks, method, keep, seed, top_k = cfg.generate(4096 * 8), 8, cfg.method, 0, cfg.seed, 0
    else:
        a = configs.planted(128, 8 * 16384, 0.0005, 64, 0.9, 1e-6, 4)
        blocks, method, keep, seed, top_k = 8, "neighbor-random", 64, 4, 64
    dm = rk.DeviceMatrix(a)
    out, _ = R.dev_full_svd(dm, blocks, method, keep, seed, True, top_k)
    try:
        res, anorm = R.dev_residual(dm, out)
        sig, u, v = R.dev_outputs_tensors(out)
        sig, u, v = sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
    finally:
        R.dev_outputs_free(out)
    k = v.shape[1]
    rep, _ = rk.repair(a, rk.partition_columns(a.cols(), blocks), method, seed)
    want, wa = dense_residual(rep, u[:, :k], sig[:k], v)
    assert abs(anorm - wa) <= 1e-12 * wa
    assert abs(res - want) <= 1e-9 * want + 1e-13 * wa, (case, res, want)
    if top_k == 0:
        assert res <= 1e-10 * anorm, (case, res / anorm)
