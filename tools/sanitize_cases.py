"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the hot path on inputs small enough for the tools.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402
from paper_2009_09767_b200.ranky import KeyedRng, RepairWorkspace  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c1"):
    # c1: ill-conditioned blocks (Householder route, TSQR), RandomChecker, V, records
    cfg = configs.CONFIGS["c1"]
    res = rk.run_pipeline(cfg.generate(), cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
    print("c1", res.svd.sigma[:3], flush=True)
if which in ("all", "c2s"):
    # a c2 slice: Gram route, cluster/DSMEM Jacobi, diag ordering, left-looking Cholesky, SYRK merge
    cfg = configs.CONFIGS["c2"]
    res = rk.run_pipeline(cfg.generate(262144 // 16), cfg.blocks // 16, cfg.method, cfg.keep, cfg.seed, 1,
                          want_v=True)
    print("c2 slice", res.svd.sigma[:3], flush=True)
if which in ("all", "nbr"):
    # NeighborChecker / NeighborRandom ordered replay (single-CTA bitmap kernel), workspace kernels
    a = configs.synth_bipartite(64, 8192, 0.002, 7)
    p = rk.partition_columns(8192, 32)
    for m in ("neighbor", "neighbor-random"):
        rep, report = rk.repair(a, p, m, 42)
        print(m, len(report.added_edges), flush=True)
    ws = RepairWorkspace(a, p)
    for d in range(4):
        for row in ws.lonely_rows(d)[:3]:
            ws.apply_neighbor_random(d, row, KeyedRng(42, d, row))
    print("workspace", ws.to_matrix().nnz(), flush=True)
if which in ("all", "dense"):
    # dense_svd (QR with V, completion), block_svd keep, metrics (Procrustes)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((48, 200))
    s = rk.dense_svd(a)
    low = rng.standard_normal((40, 5)) @ rng.standard_normal((5, 30))
    rk.dense_svd(low)
    print("dense", s.sigma[:2], rk.numerical_rank(low, 1e-10), rk.left_vector_error(s.u, s.u, s.sigma), flush=True)
if which in ("all", "c3s"):
    # a c3 slice: wide blocks on the reduced route (QR with T kept, the shared-memory Gram-assisted Jacobi at
    # cluster sizes 1 and 2, the compact-WY apply_q), NeighborChecker, eigensolver merge
    cfg = configs.CONFIGS["c3"]
    res = rk.run_pipeline(cfg.generate(8192 * 16), 16, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
    print("c3 slice", res.svd.sigma[:3], flush=True)
if which in ("all", "wide"):
    # a c4 slice: 1024-row Gram-route blocks through the wide pair-block Jacobi (one launch per step)
    cfg = configs.CONFIGS["c4"]
    res = rk.run_pipeline(cfg.generate(16384 * 2), 2, cfg.method, cfg.keep, cfg.seed, 1, want_v=False)
    print("c4 slice", res.svd.sigma[:3], flush=True)
