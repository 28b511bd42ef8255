"""Generate tests/golden/{c4,c5}_merge_reference.npz: SURVEY.md §8(c)(iii) for the
configs whose full CPU run is infeasible.

The GPU's own per-block records (rk_run_pipeline, the same records the device
merge consumes) are fed into the unmodified reference's proxy_from_records +
proxy_svd (proj/src/pipeline.cpp:18-59, proj/src/proxy.cpp:40-46, through
oracle/_ref/libranky_ref.so). The reference's final sigma and U are the golden;
tests/test_gpu_scale.py checks the device pipeline's sigma and U against them at
the north_star tolerances. V: recover_right_vectors (proj/src/proxy.cpp:48-72)
of the reference on one block of columns of the repaired matrix with the
reference's U and sigma.

Needs a GPU and the reference build; runs on the GPU box (c4: ~30 min of
single-threaded reference proxy_svd). c5's full proxy_svd (~1.5 h) outlasts one
GPU-box call, so for c5 P is first reduced to R^T (M x M) by a LAPACK Householder QR
of P^T -- an orthogonal right factor: sigma and U unchanged -- and the reference's
proxy_from_records + proxy_svd run on that (--reduce):

    python tests/golden/make_merge_golden.py c4
    python tests/golden/make_merge_golden.py c5 tests/golden 0 --reduce
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Oracle  # noqa: E402
from paper_2009_09767_b200 import configs  # noqa: E402
import paper_2009_09767_b200 as rk  # noqa: E402

U_COLS = {"c4": 256, "c5": 64}   # U columns stored (c5 is a top-64 config)
V_BLOCK = {"c4": 613, "c5": 2901}
V_COLS = 512


def main(name, out_dir, scale=None, reduce=False):
    t0 = time.perf_counter()

    def mark(what):
        print(f"[{name}] {what}: {time.perf_counter() - t0:.1f} s", flush=True)

    R = Oracle("reference")
    cfg = configs.CONFIGS[name]
    if scale:  # dry run: the config's block width, scale // width blocks
        import dataclasses
        cfg = dataclasses.replace(cfg, cols=scale, blocks=scale // (cfg.cols // cfg.blocks))
    a = cfg.generate(scale)
    M = a.rows()
    mark("generated")
    res = rk.run_pipeline(a, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=False, top_k=cfg.top_k,
                          want_repaired=True, want_records=True)
    mark(f"GPU pipeline ({res.timing['total_ms'] / 1e3:.1f} s device)")
    del a
    k = U_COLS[name]
    gpu_sigma, gpu_u = np.array(res.svd.sigma), np.array(res.svd.u[:, :k])
    recs = [np.asarray(r.payload).reshape(r.rows, r.kept) for r in res.records]
    res.records.clear()
    rep = res.repaired
    np.savez_compressed(os.path.join(out_dir, f"{name}_merge_gpu.npz"), sigma=gpu_sigma, u=gpu_u)
    if reduce:
        # P (M x sum k) -> R^T (M x M) by a LAPACK Householder QR of P^T: an orthogonal
        # right factor, so sigma and U are unchanged (backward stable); the reference's
        # proxy_from_records + proxy_svd then run on R^T as one record. For c5, whose
        # full single-threaded proxy_svd (~1.5 h) outlasts one GPU-box call.
        pt = np.concatenate(recs, axis=1).T.copy()
        del recs
        r = np.linalg.qr(pt, mode="r")
        del pt
        mark(f"LAPACK QR of P^T ({r.shape})")
        recs = [np.ascontiguousarray(r.T)]
    o = R.proxy_svd_records(recs)
    del recs
    mark("reference proxy_from_records + proxy_svd" + (" on R^T" if reduce else ""))
    p = rk.partition_columns(rep.cols(), cfg.blocks)
    rng = p.range(min(V_BLOCK[name], cfg.blocks - 1))
    lo = rng.begin
    rr, rc, rv = rep.coo()
    m = (rc >= lo) & (rc < lo + V_COLS)
    kk = cfg.top_k or len(o.sigma)
    vs = R.recover_right_vectors((M, V_COLS, rr[m], rc[m] - lo, rv[m]), o.u[:, :kk], o.sigma[:kk], 1e-10)
    np.savez_compressed(os.path.join(out_dir, f"{name}_merge_reference.npz"), sigma=o.sigma, u=o.u[:, :k],
                        v_rows=vs, v_begin=np.int64(lo), records_from="GPU rk_run_pipeline records",
                        reduced_by_lapack_qr=np.bool_(reduce),
                        proxy_s=np.float64(time.perf_counter() - t0))
    rel = np.abs(gpu_sigma - o.sigma[:len(gpu_sigma)]) / o.sigma[:len(gpu_sigma)]
    mark(f"done; GPU vs reference sigma max rel {rel[o.sigma[:len(gpu_sigma)] > 1e-10 * o.sigma[0]].max():.2e}")


if __name__ == "__main__":
    # optional 3rd argument: a reduced column count (a multiple of the block count) for a dry
    # run (0: full size); --reduce: P -> R^T by LAPACK QR before the reference's proxy_svd
    args = [a for a in sys.argv[1:] if a != "--reduce"]
    main(args[0], args[1] if len(args) > 1 else HERE, int(args[2]) if len(args) > 2 and int(args[2]) else None,
         "--reduce" in sys.argv)
