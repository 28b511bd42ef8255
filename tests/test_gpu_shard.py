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
from parity import compare

pytestmark = pytest.mark.gpu


def run_sharded(dm, cfg, world, route="tsqr"):
    """route "tsqr": rk_dev_shard_factor + rk_dev_shard_finish. route "gram": the
    protocol of bench.py -- rk_dev_shard_factor_gram, all-gather of the Gram
    partials, rk_dev_shard_finish_gram, with the TSQR fallback when either call
    returns RK_GRAM_REJECTED. Returns the outputs and whether the Gram route held."""
    import torch
    L = R.lib()
    M = cfg.rows
    plans = [shard.plan(M, cfg.cols if dm.cols == cfg.cols else dm.cols, cfg.blocks, cfg.keep, world, g)
             for g in range(world)]
    roots = torch.empty((world, M, M), dtype=torch.float64, device="cuda")
    handles = []
    gram = route == "gram"
    for g, sp in enumerate(plans):
        h = C.c_void_p()
        t = R.Timing()
        args = (dm.ctx.handle, dm.handle, cfg.blocks, R._method(cfg.method), cfg.keep, cfg.seed, sp.leaf_lo,
                sp.leaf_hi, C.c_void_p(roots[g].data_ptr()), C.byref(h), C.byref(t))
        st = L.rk_dev_shard_factor_gram(*args) if gram else R.GRAM_REJECTED
        if st == R.GRAM_REJECTED:
            assert g == 0 or not gram, "the Gram route's applicability must not depend on the rank"
            gram = False
            st = L.rk_dev_shard_factor(*args)
        R._check(st)
        handles.append(h)
    dm.ctx.synchronize()
    outs = []
    rejected = False
    for g, sp in enumerate(plans):
        out = C.POINTER(R.DevOutputs)()
        t = R.Timing()
        args = (dm.ctx.handle, handles[g], C.c_void_p(roots.data_ptr()), world, R.WANT_V, cfg.top_k, sp.col_lo,
                sp.col_hi, C.byref(out), C.byref(t))
        if gram:
            st = L.rk_dev_shard_finish_gram(*args)
            if st == R.GRAM_REJECTED:
                assert g == 0 or rejected, "the kappa guard must decide identically on every rank"
                rejected = True
                break
            R._check(st)
        else:
            R._check(L.rk_dev_shard_finish(*args))
        sig, u, v = R.dev_outputs_tensors(out)
        outs.append((sp, sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()))
        R.dev_outputs_free(out)
    if rejected:  # every rank: its TSQR factor, all-gather, the TSQR finish
        gram = False
        for g in range(world):
            R._check(L.rk_dev_shard_tsqr(dm.ctx.handle, handles[g], C.c_void_p(roots[g].data_ptr())))
        dm.ctx.synchronize()
        for g, sp in enumerate(plans):
            out = C.POINTER(R.DevOutputs)()
            t = R.Timing()
            R._check(L.rk_dev_shard_finish(dm.ctx.handle, handles[g], C.c_void_p(roots.data_ptr()), world,
                                           R.WANT_V, cfg.top_k, sp.col_lo, sp.col_hi, C.byref(out), C.byref(t)))
            sig, u, v = R.dev_outputs_tensors(out)
            outs.append((sp, sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()))
            R.dev_outputs_free(out)
    for h in handles:
        L.rk_dev_shard_destroy(h)
    return (outs, gram) if route == "gram" else outs


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


@pytest.mark.parametrize("name", ["c2", "c1"])
def test_sharded_gram_route(name):
    """The Gram route of the sharded merge: bitwise identical for every G (the
    ranks' partials are nodes of one pairwise tree), parity with the single-GPU
    call; c1's merge (kappa > kappa_max) exercises the rejection and the TSQR
    fallback, which must then equal the TSQR route bitwise."""
    cfg = configs.CONFIGS[name]
    a = cfg.generate()
    dm = rk.DeviceMatrix(a)
    out, _ = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    sig, u, v = R.dev_outputs_tensors(out)
    sig, u, v = sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
    R.dev_outputs_free(out)
    n_leaves = shard.merge_tree_leaves(cfg.rows, a.cols(), cfg.blocks, cfg.keep)
    ref = None
    for world in (1, 2, 4, 8):
        if world > n_leaves or not shard.bitwise_invariant(n_leaves, world):
            continue
        outs, held = run_sharded(dm, cfg, world, "gram")
        if ref is None:
            ref = outs[0]
            compare(SimpleNamespace(sigma=ref[1], u=ref[2]), sig, u, f"{name} gram shard(1) vs single")
            if not held:  # rejected: the fallback is the TSQR route exactly
                [(_, s_t, u_t, v_t)] = run_sharded(dm, cfg, 1)
                assert np.array_equal(s_t, ref[1]) and np.array_equal(u_t, ref[2])
        for sp, s2, u2, v2 in outs:
            assert np.array_equal(s2, ref[1]) and np.array_equal(u2, ref[2]), (name, world, sp.rank)
            assert np.array_equal(v2, ref[3][sp.col_lo:sp.col_hi]), (name, world, sp.rank)
    if name == "c2":
        assert held, "c2's merge is well conditioned: the Gram route must hold"


def test_sharded_gram_not_applicable(tuning_env):
    """RK_BLOCK_ROUTE=householder turns the Gram routes off: factor_gram reports
    RK_GRAM_REJECTED (no shard) and the protocol takes the TSQR path."""
    tuning_env("RK_BLOCK_ROUTE", "householder")
    cfg = configs.CONFIGS["c1"]
    dm = rk.DeviceMatrix(cfg.generate())
    outs, held = run_sharded(dm, cfg, 2, "gram")
    assert not held
    tsqr = run_sharded(dm, cfg, 2)
    for (sp, s1, u1, v1), (_, s2, u2, v2) in zip(outs, tsqr):
        assert np.array_equal(s1, s2) and np.array_equal(u1, u2) and np.array_equal(v1, v2)
