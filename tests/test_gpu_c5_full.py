"""c5 at full size (M=2048, N=67,108,864, 4096 blocks, ~68.7M nnz, keep 64, top-64),
in the default GPU pass.

The reference cannot run c5 (~250 h of block work), so parity follows
SURVEY.md §8(c):
  (i)   repair in full, bit-exact against the reference's ranky::repair;
  (ii)  one sampled block against the reference's block_svd (keep 64), computed on
        the host while the device pipeline runs;
  (iii) the final sigma and U against the reference's proxy_from_records + proxy_svd
        on the GPU's own block records (tests/golden/c5_merge_reference.npz, made by
        tests/golden/make_merge_golden.py: P reduced to R^T by a LAPACK QR first);
  (iv)  V: a block of rows bit-exact against recover_right_vectors given our U and
        sigma, the golden's rows (the reference's U and sigma) to 1e-6 relative, and
        V's 64 columns orthonormal over all N rows up to the keep-64 truncation.
"""
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200.ranky import dev_outputs_tensors, dev_residual
from parity import check_sigma, check_u, check_v_rows, compare
from test_gpu_scale import coo_of, load_golden

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.timeout(3600)
def test_c5_full_size(ref):
    import torch
    gold = load_golden("c5")
    if gold is None:
        pytest.skip("tests/golden/c5_merge_reference.npz not generated")
    t0 = time.perf_counter()

    def mark(what):
        print(f"[c5] {what}: {time.perf_counter() - t0:.1f} s", flush=True)

    cfg = configs.CONFIGS["c5"]
    a = cfg.generate()
    M, N = a.rows(), a.cols()
    mark(f"generated {a.nnz()} nnz")
    p = rk.partition_columns(N, cfg.blocks)
    rep, report = rk.repair(a, p, cfg.method, cfg.seed)
    mark(f"repaired on the device ({len(report.added_edges)} edges, {report.fallback_count} fallbacks)")
    ex = ThreadPoolExecutor(2)  # the reference's pieces run on the host while the device works
    f_rep = ex.submit(lambda: ref.repair(coo_of(a), cfg.blocks, cfg.method, cfg.seed))
    d_blk = cfg.blocks // 2 + 17
    view = rk.block_view(rep, p, d_blk)
    f_blk = ex.submit(lambda: ref.block_svd(coo_of(view), cfg.keep))

    dm = rk.DeviceMatrix(a)
    out, t = rk.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    mark(f"device pipeline: {t.total_ms / 1e3:.1f} s (blocks {t.blocks_ms / 1e3:.1f} = QR {t.qr_ms / 1e3:.1f} + "
         f"Jacobi {t.jacobi_ms / 1e3:.1f}; merge {t.merge_ms / 1e3:.1f}, V {t.recover_ms / 1e3:.1f})")
    try:
        sig_d, u_d, v_d = dev_outputs_tensors(out)
        sigma, u = sig_d.cpu().numpy(), u_d.cpu().numpy()
        k = cfg.top_k
        # (iii) against the reference's merge of our records
        worst = check_sigma(sigma, gold["sigma"], "c5 sigma vs reference")
        ov, sn = check_u(u, gold["u"], gold["sigma"], "c5 U vs reference", cols=k)
        mark(f"sigma/U vs reference: sigma rel {worst:.2e}, min signed overlap 1-{1 - ov:.1e}, cluster sin {sn:.1e}")
        # (iv) V
        assert tuple(v_d.shape) == (N, k)
        lo = int(gold["v_begin"])
        vg = gold["v_rows"]
        check_v_rows(v_d[lo:lo + vg.shape[0]].cpu().numpy(), vg, gold["sigma"][:k], "c5 V rows vs reference")
        d = 1234
        rng_d = p.range(d)
        vr = ref.recover_right_vectors(coo_of(rk.block_view(rep, p, d)), u[:, :k], sigma[:k], rk.K_RANK_TOL)
        assert np.array_equal(v_d[rng_d.begin:rng_d.end].cpu().numpy(), vr)
        vtv = torch.zeros(k, k, dtype=torch.float64, device=v_d.device)
        step = 1 << 22
        for r0 in range(0, N, step):
            blk = v_d[r0:r0 + step]
            vtv += blk.T @ blk
        orth = float((vtv - torch.eye(k, dtype=torch.float64, device=v_d.device)).abs().max())
        res, anorm = dev_residual(dm, out)
        mark(f"V orthonormality {orth:.2e}; residual/||A|| {res / anorm:.6e}")
        # keep = 64 per block: P P^T is A A^T minus the blocks' tails, so V = A^T U Sigma^-1
        # is orthonormal only up to that truncation (the reference's algorithm)
        assert orth <= 1e-5
        # U_k Sigma_k V^T = U_k U_k^T A (V = A^T U Sigma^-1), so res^2 = ||A||^2 - ||U_k^T A||^2, and
        # ||A^T u_j|| >= ||P^T u_j|| = sigma_j (P P^T <= A A^T): res <= sqrt(||A||^2 - sum sigma_j^2)
        bound = np.sqrt(max(0.0, anorm ** 2 - float(np.sum(sigma[:k] ** 2))))
        assert res <= bound * (1 + 1e-9) + 1e-12 * anorm, (res, bound, anorm)
    finally:
        rk.dev_outputs_free(out)
        dm.close()
    # (i), (ii)
    o = f_rep.result()
    assert np.array_equal(report.edges_array(), o.edges)
    assert report.lonely_counts == o.lonely_counts.tolist()
    assert report.fallback_count == o.fallback_count
    rr, rc, rv = rep.coo()
    assert np.array_equal(rr, o.matrix[2]) and np.array_equal(rc, o.matrix[3]) and np.array_equal(rv, o.matrix[4])
    mark("repair bit-exact")
    want = f_blk.result()
    compare(rk.block_svd(view, cfg.keep), want.sigma, want.u, f"c5 block {d_blk}")
    mark("sampled block")
    ex.shutdown()
