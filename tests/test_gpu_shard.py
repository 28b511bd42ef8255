"""The sharded entry points (rk_dev_shard_factor / rk_dev_shard_finish), on one
GPU: G ranks are run one after another in this process (no rank waits on
another), their subtree factors gathered into one buffer as the NCCL all-gather
of bench.py would, and every rank's finish compared. With leaves / G a power of
two every rank's factor is a node of the one-rank tree, so sigma and U are
bitwise identical for every G and a rank's V rows are bitwise the one-rank V
rows of its columns; against the single-GPU rk_dev_full_svd (whose merge may
take the Gram route) the agreement is the parity tolerance."""
import ctypes as C
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs, shard
from paper_2009_09767_b200 import ranky as R
from test_gpu_svd import compare

pytestmark = pytest.mark.gpu


def run_sharded(dm, cfg, world):
    import torch
    L = R.lib()
    M = cfg.rows
    plans = [shard.plan(M, cfg.cols if dm.cols == cfg.cols else dm.cols, cfg.blocks, cfg.keep, world, g)
             for g in range(world)]
    roots = torch.empty((world, M, M), dtype=torch.float64, device="cuda")
    handles = []
    for g, sp in enumerate(plans):
        h = C.c_void_p()
        t = R.Timing()
        R._check(L.rk_dev_shard_factor(dm.ctx.handle, dm.handle, cfg.blocks, R._method(cfg.method), cfg.keep,
                                       cfg.seed, sp.leaf_lo, sp.leaf_hi, C.c_void_p(roots[g].data_ptr()),
                                       C.byref(h), C.byref(t)))
        handles.append(h)
    dm.ctx.synchronize()
    outs = []
    for g, sp in enumerate(plans):
        out = C.POINTER(R.DevOutputs)()
        t = R.Timing()
        R._check(L.rk_dev_shard_finish(dm.ctx.handle, handles[g], C.c_void_p(roots.data_ptr()), world, R.WANT_V,
                                       cfg.top_k, sp.col_lo, sp.col_hi, C.byref(out), C.byref(t)))
        sig, u, v = R.dev_outputs_tensors(out)
        outs.append((sp, sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()))
        R.dev_outputs_free(out)
        L.rk_dev_shard_destroy(handles[g])
    return outs


@pytest.mark.parametrize("name,scale", [("c2", None), ("c1", None)])
def test_sharded_matches_single_gpu(name, scale):
    cfg = configs.CONFIGS[name]
    a = cfg.generate(scale)
    dm = rk.DeviceMatrix(a)
    out, _ = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    sig, u, v = R.dev_outputs_tensors(out)
    sig, u, v = sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
    R.dev_outputs_free(out)
    # one rank: the TSQR merge tree (the single-GPU call may take the Gram route
    # for the merge, so it agrees to rounding, not bitwise)
    [(sp1, s1, u1, v1)] = run_sharded(dm, cfg, 1)
    compare(SimpleNamespace(sigma=s1, u=u1), sig, u, f"{name} shard(1) vs single")
    cos = np.sum(v1 * v, axis=0) / (np.linalg.norm(v1, axis=0) * np.linalg.norm(v, axis=0))
    assert np.all(np.abs(cos) >= 1 - 1e-8)
    n_leaves = shard.merge_tree_leaves(cfg.rows, a.cols(), cfg.blocks, cfg.keep)
    for world in (2, 4, 8):
        if world > n_leaves:
            continue
        outs = run_sharded(dm, cfg, world)
        exact = shard.bitwise_invariant(n_leaves, world)
        for sp, s2, u2, v2 in outs:
            if exact:
                assert np.array_equal(s2, s1) and np.array_equal(u2, u1), (name, world, sp.rank)
                assert np.array_equal(v2, v1[sp.col_lo:sp.col_hi]), (name, world, sp.rank)
            else:
                assert np.allclose(s2, s1, rtol=1e-10, atol=0), (name, world, sp.rank)
        # the ranks' V rows tile the matrix's columns
        assert sum(sp.col_hi - sp.col_lo for sp, *_ in outs) == a.cols()
