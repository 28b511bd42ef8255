"""The sharded (one process per GPU) orchestration on CPU with torch.distributed
gloo, world size 2: shard plans cover every leaf and column exactly once, and
gathering per-rank subtree factors then finishing the fixed pairwise tree gives
bitwise the same factor as the single-process tree. The per-node QR here is
numpy (a stand-in for the CUDA kernels, which need a GPU); what is tested is the
plan, the all-gather order and the tree shape bench.py and
rk_dev_shard_factor / rk_dev_shard_finish rely on."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_09767_b200 import shard


def test_plan_covers_everything():
    for (rows, cols, blocks, keep) in [(256, 262144, 64, 0), (64, 8192, 16, 0), (2048, 67108864, 4096, 64),
                                       (16, 100, 7, 0)]:
        leaves = shard.leaf_blocks(rows, cols, blocks, keep)
        assert leaves[0][0] == 0 and leaves[-1][1] == blocks
        assert all(a[1] == b[0] for a, b in zip(leaves, leaves[1:]))
        for world in (1, 2, 4, 8):
            if world > len(leaves):
                continue
            plans = [shard.plan(rows, cols, blocks, keep, world, g) for g in range(world)]
            assert plans[0].leaf_lo == 0 and plans[-1].leaf_hi == len(leaves)
            assert plans[0].col_lo == 0 and plans[-1].col_hi == cols
            for p, q in zip(plans, plans[1:]):
                assert p.leaf_hi == q.leaf_lo and p.col_hi == q.col_lo


def test_plan_matches_library_leaf_count():
    for args in [(256, 262144, 64, 0), (64, 8192, 16, 0), (2048, 67108864, 4096, 64), (512, 4194304, 512, 0)]:
        assert shard.merge_tree_leaves(*args) == len(shard.leaf_blocks(*args))
    assert shard.bitwise_invariant(64, 8) and not shard.bitwise_invariant(48, 8)


def _r_of(stack):
    r = np.linalg.qr(stack, mode="r")
    return r * np.sign(np.diag(r))[:, None]  # canonical signs: deterministic factor


def _leaf_factors(seed, n_leaves, m):
    rng = np.random.default_rng(seed)
    return [_r_of(rng.standard_normal((m + 3, m))) for _ in range(n_leaves)]


def _combine(a, b):
    return _r_of(np.vstack([a, b]))


def _worker(rank, world, port, n_leaves, m, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        leaves = _leaf_factors(7, n_leaves, m)
        per = n_leaves // world
        mine = shard.pairwise_tree(leaves[rank * per:(rank + 1) * per], _combine)
        gathered = [torch.zeros(m, m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(mine)))
        root = shard.pairwise_tree([g.numpy() for g in gathered], _combine)
        q.put((rank, root))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_gloo_world2_matches_single_tree():
    n_leaves, m = 8, 12
    single = shard.pairwise_tree(_leaf_factors(7, n_leaves, m), _combine)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_leaves, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for _, root in results:
        assert np.array_equal(root, single)
