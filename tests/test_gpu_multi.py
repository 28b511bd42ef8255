"""Library-owned multi-GPU runs (rk_multi_*, rk_dev_sharded_full_svd), on one GPU.

* rk_multi_run_pipeline with devices [0, 0] / [0, 0, 0, 0]: the shards run
  concurrently on threads of this process and exchange their factors by device
  copies (peer copies between distinct devices); the result equals the
  single-GPU run_pipeline to the parity tolerance and is bitwise the same for 2
  and 4 shards; report, repaired matrix and records equal the single run's.
* rk_dev_sharded_full_svd from two processes (torch.multiprocessing, gloo) sharing
  device 0: the library orchestrates factor -> all-gather -> finish, the caller's
  all-gather is gloo on host copies. Each rank's sigma / U equal the 2-shard
  rk_multi result bitwise, its V rows the same rows of it.
Kernels of different shards never wait on one another: the exchange is host
synchronised after every shard's factor is complete."""
import os
import socket

import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200 import ranky as R
from parity import compare

pytestmark = pytest.mark.gpu


def _c2_slice(nb=16):
    cfg = configs.CONFIGS["c2"]
    cols = 262144 * nb // cfg.blocks
    return cfg, cfg.generate(cols), nb


@pytest.mark.parametrize("name", ["c1", "c2s"])
def test_multi_matches_single(name, ref):
    if name == "c1":
        cfg = configs.CONFIGS["c1"]
        a, D = cfg.generate(), cfg.blocks
    else:
        cfg, a, D = _c2_slice()
    single = rk.run_pipeline(a, D, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
    outs = []
    for devs in ([0, 0], [0, 0, 0, 0]):
        m = R.Multi(devs)
        try:
            res = m.run_pipeline(a, D, cfg.method, cfg.keep, cfg.seed, want_v=True)
        finally:
            m.close()
        compare(res.svd, single.svd.sigma, single.svd.u, f"{name} multi {devs}")
        assert res.report.edges_array().tolist() == single.report.edges_array().tolist()
        assert res.report.lonely_counts == single.report.lonely_counts
        assert res.repaired == single.repaired
        assert len(res.records) == len(single.records)
        for x, y in zip(res.records, single.records):
            assert x == y, f"record {x.block_index} differs"
        r, c, v = res.repaired.coo()
        vr = ref.recover_right_vectors((a.rows(), a.cols(), r, c, v), res.svd.u, res.svd.sigma, 1e-10)
        assert np.array_equal(res.svd.v, vr)
        outs.append(res)
    assert np.array_equal(outs[0].svd.sigma, outs[1].svd.sigma) and np.array_equal(outs[0].svd.u, outs[1].svd.u)
    assert np.array_equal(outs[0].svd.v, outs[1].svd.v)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg, a, D = _c2_slice()
        ctx = rk.Context(0)
        dm = rk.DeviceMatrix(a, ctx)

        def allgather(mine, alls):  # gloo on host copies, rank order
            parts = [torch.empty(mine.numel(), dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, mine.cpu())
            alls.copy_(torch.cat(parts).to(alls.device))
            torch.cuda.synchronize()

        out, t, lo, hi = R.dev_sharded_full_svd(dm, D, cfg.method, cfg.keep, cfg.seed, world, rank, allgather)
        sig, u, v = R.dev_outputs_tensors(out)
        q.put((rank, sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy(), lo, hi, int(t.kernel_launches)))
        R.dev_outputs_free(out)
        dm.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo_library_orchestration():
    import torch.multiprocessing as mp
    cfg, a, D = _c2_slice()
    m = R.Multi([0, 0])
    try:
        want = m.run_pipeline(a, D, cfg.method, cfg.keep, cfg.seed, want_v=True)
    finally:
        m.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    for rank, sig, u, v, lo, hi, launches in got:
        assert launches > 0
        assert np.array_equal(sig, want.svd.sigma) and np.array_equal(u, want.svd.u)
        assert np.array_equal(v, want.svd.v[lo:hi])
    assert sorted((lo, hi) for _, _, _, _, lo, hi, _ in got)[0][0] == 0
