"""GPU evaluation metrics (rk_eval.cu) against the reference's own
proj/src/metrics.cpp:32-114 (sigma_error, align_signs with sign flips and
Procrustes on degenerate clusters, left_vector_error, numerical_rank)."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk

pytestmark = pytest.mark.gpu


def orthonormal(rng, m, n):
    q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    return q


def test_sigma_error(ref):
    rng = np.random.default_rng(3)
    for na, nb in [(5, 5), (3, 7), (9, 2), (0, 4), (1000, 1000)]:
        a, b = rng.uniform(0, 2, na), rng.uniform(0, 2, nb)
        want = ref.sigma_error(a, b) if ref.kind == "reference" else float(
            np.abs(np.pad(a, (0, max(0, nb - na))) - np.pad(b, (0, max(0, na - nb)))).sum())
        assert abs(rk.sigma_error(a, b) - want) <= 1e-13 * max(1.0, want)


@pytest.mark.parametrize("with_sigma", [False, True])
def test_align_signs_and_left_vector_error(ref, with_sigma):
    if ref.kind != "reference":
        pytest.skip("needs the reference build (oracle/_ref)")
    rng = np.random.default_rng(5)
    m, n = 40, 12
    u = orthonormal(rng, m, n)
    sigma = np.array([9, 8, 8, 8, 7, 6, 5, 5, 4, 3, 2, 1], dtype=float)
    # u_hat: columns flipped and the degenerate clusters rotated inside their span
    hat = u * np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
    for lo, hi in [(1, 4), (6, 8)]:
        q = orthonormal(rng, hi - lo, hi - lo)
        hat[:, lo:hi] = hat[:, lo:hi] @ q
    hat += 1e-9 * rng.standard_normal(hat.shape)
    sg = sigma if with_sigma else None
    got = rk.align_signs(hat, u, sg)
    want = ref.align_signs(hat, u, sg)
    assert np.max(np.abs(got - want)) <= 1e-12
    if with_sigma:
        assert np.max(np.abs(got - u)) <= 1e-8
        e = rk.left_vector_error(hat, u, sigma)
        assert abs(e - ref.left_vector_error(hat, u, sigma)) <= 1e-12 * max(1.0, e)
        assert e <= 1e-6
    with pytest.raises(rk.InvalidArgument):
        rk.align_signs(hat, u, sigma[:5])
    with pytest.raises(rk.InvalidArgument):
        rk.align_signs(hat[:, :3], u)


def test_numerical_rank(ref):
    rng = np.random.default_rng(9)
    for m, n, r in [(20, 30, 7), (30, 20, 20), (16, 16, 1), (8, 5, 0)]:
        a = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) if r else np.zeros((m, n))
        got = rk.numerical_rank(a, 1e-10)
        assert got == r
        if ref.kind == "reference":
            assert got == ref.numerical_rank(a, 1e-10)


def test_device_forms_on_pipeline_outputs():
    """left_vector_error / sigma_error on device tensors: a pipeline's U against itself
    with flipped signs is exactly aligned back (error 0)."""
    import torch
    from paper_2009_09767_b200 import configs
    from paper_2009_09767_b200.ranky import dev_left_vector_error, dev_sigma_error, dev_outputs_tensors
    cfg = configs.CONFIGS["c1"]
    dm = rk.DeviceMatrix(cfg.generate())
    out, _ = rk.ranky.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, False, 0)
    try:
        sig, u, _ = dev_outputs_tensors(out)
        flipped = u * torch.where(torch.arange(u.shape[1], device=u.device) % 2 == 0, -1.0, 1.0).double()
        assert dev_left_vector_error(flipped.contiguous(), u.contiguous(), sig.contiguous()) <= 1e-13
        assert dev_sigma_error(sig, sig) == 0.0
    finally:
        rk.ranky.dev_outputs_free(out)
        dm.close()
