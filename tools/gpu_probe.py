"""Quick GPU probe used while developing: runs each kernel family once against
the CPU oracles and prints the worst errors. Not collected by pytest."""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2009_09767_b200 as rk  # noqa: E402
from paper_2009_09767_b200 import configs as cf  # noqa: E402
from oracle import Oracle, available  # noqa: E402

REF = Oracle("reference") if available("reference") else Oracle("port")
print("oracle kind:", REF.kind, flush=True)


def coo(a):
    r, c, v = a.coo()
    return (a.rows(), a.cols(), r, c, v)


def step(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time() - t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def t_rng():
    out = rk.keyed_rng_next(0, [0], [0], 3)[0]
    ref = REF.rng_stream(0, 0, 0, 3)
    assert np.array_equal(out, ref), (out, ref)
    b = rk.keyed_rng_below(42, [0], [8], [1024])[0]
    assert b == 587, b


def t_repair():
    for seed in range(3):
        a = cf.synth_bipartite(16, 128, 0.05, seed)
        for D in (1, 3, 8):
            for m in ("random", "neighbor", "neighbor-random", "none"):
                rep, report = rk.repair(a, rk.partition_columns(128, D), m, seed + 5)
                ref = REF.repair(coo(a), D, m, seed + 5)
                assert np.array_equal(report.edges_array().reshape(-1, 4), ref.edges.reshape(-1, 4)), (seed, D, m)
                assert list(report.lonely_counts) == list(ref.lonely_counts)
                assert report.fallback_count == ref.fallback_count
                rr, rc, rv = rep.coo()
                assert np.array_equal(rr, ref.matrix[2]) and np.array_equal(rc, ref.matrix[3])
                assert np.array_equal(rv, ref.matrix[4])
    a = cf.CONFIGS["c1"].generate()
    rep, report = rk.repair(a, rk.partition_columns(a.cols(), 16), "neighbor-random", 0)
    ref = REF.repair(coo(a), 16, "neighbor-random", 0)
    assert np.array_equal(report.edges_array(), ref.edges)


def cmp_svd(name, s, ref, tol_rel=1e-10):
    sig, rsig = np.asarray(s.sigma), np.asarray(ref.sigma)
    assert sig.shape == rsig.shape, (sig.shape, rsig.shape)
    smax = rsig.max() if len(rsig) else 0
    big = rsig > 1e-8 * smax
    rel = np.max(np.abs(sig[big] - rsig[big]) / rsig[big]) if big.any() else 0
    absd = np.max(np.abs(sig - rsig)) / max(smax, 1e-300) if len(rsig) else 0
    # overlaps of non-degenerate columns
    ov = 1.0
    for j in range(len(rsig)):
        if not big[j]:
            continue
        gap = min(abs(rsig[j] - rsig[j - 1]) if j else np.inf, abs(rsig[j] - rsig[j + 1]) if j + 1 < len(rsig) else np.inf)
        if gap <= 1e-9 * smax:
            continue
        ov = min(ov, abs(float(s.u[:, j] @ ref.u[:, j])))
    print(f"    {name}: sigma rel {rel:.2e} abs/smax {absd:.2e} min overlap 1-{1 - ov:.1e}")
    assert rel <= tol_rel and 1 - ov <= 1e-8, (rel, ov)


def t_dense():
    rng = np.random.default_rng(0)
    for shape in [(2, 2), (14, 14), (6, 40), (40, 6), (16, 256), (64, 64), (100, 300), (300, 100)]:
        a = rng.uniform(-1, 1, shape)
        s = rk.dense_svd(a)
        ref = REF.dense_svd(a)
        cmp_svd(f"dense {shape}", s, ref)
        orth = np.abs(s.u.T @ s.u - np.eye(s.u.shape[1])).max()
        orthv = np.abs(s.v.T @ s.v - np.eye(s.v.shape[1])).max()
        resid = np.linalg.norm(a - s.u @ np.diag(s.sigma) @ s.v.T) / max(1, np.linalg.norm(a))
        print(f"      orth U {orth:.1e} V {orthv:.1e} resid {resid:.1e}")
        assert orth < 1e-10 and orthv < 1e-10 and resid < 1e-10
    s = rk.dense_svd(np.array([[0, 0, 0, 0], [6.0, 0, 0, 8.0]]))
    print("    rank-1:", s.sigma)


def t_block():
    for seed in range(3):
        for (m, n, dens) in [(64, 512, 0.01), (16, 256, 0.5), (9, 4, 1.0), (256, 4096, 0.005), (64, 64, 0.3)]:
            a = cf.uniform(m, n, dens, cf.VAL_UNIFORM_PM1, seed)
            s = rk.block_svd(a, m)
            ref = REF.block_svd(coo(a), m)
            cmp_svd(f"block {m}x{n} d={dens}", s, ref)


def t_recover():
    a = cf.uniform(32, 2000, 0.05, cf.VAL_NORMAL, 3)
    ref = REF.dense_svd(a.to_dense())
    v = rk.recover_right_vectors(a, ref.u, ref.sigma, 1e-10)
    vr = REF.recover_right_vectors(coo(a), ref.u, ref.sigma, 1e-10)
    assert v.shape == vr.shape and np.array_equal(v, vr), np.abs(v - vr).max()


def t_pipeline(name, scale=None):
    c = cf.CONFIGS[name]
    a = c.generate(scale)
    t = time.time()
    res = rk.run_pipeline(a, c.blocks, c.method, c.keep, c.seed, 1, want_v=True)
    t1 = time.time()
    ref = REF.full_svd(coo(a), c.blocks, c.method, c.keep, c.seed, os.cpu_count() or 1)
    t2 = time.time()
    print(f"    gpu {t1 - t:.3f}s cpu-ref {t2 - t1:.3f}s timing {res.timing}")
    cmp_svd(f"pipeline {name}", res.svd, ref)
    vv = res.svd.v
    assert vv.shape == ref.v.shape
    ov = np.min(np.abs(np.sum(vv * ref.v, axis=0)) / (np.linalg.norm(vv, axis=0) * np.linalg.norm(ref.v, axis=0)))
    print(f"    V min |cos| 1-{1 - ov:.1e}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "repair", "dense", "block", "recover", "c1", "c2"]
    if "rng" in which: step("rng", t_rng)
    if "repair" in which: step("repair", t_repair)
    if "dense" in which: step("dense", t_dense)
    if "block" in which: step("block", t_block)
    if "recover" in which: step("recover", t_recover)
    if "c1" in which: step("pipeline c1", lambda: t_pipeline("c1"))
    if "c2" in which: step("pipeline c2", lambda: t_pipeline("c2"))
    if "c3s" in which: step("pipeline c3 (N/16)", lambda: t_pipeline("c3", 4194304 // 16))
