"""Parity rules shared by every GPU test (BASELINE.json north_star).

* singular values: relative error <= 1e-10 for sigma_ref > 1e-10·sigma_max;
  absolute <= 1e-8·sigma_max below that split (exact-zero sigma of
  rank-deficient blocks);
* singular vectors: clusters are formed as the reference's metrics do
  (consecutive sigma_ref within 1e-9·sigma_max, proj/src/metrics.cpp:15,63-70).
  A singleton column must match the reference **with its sign**:
  <u, u_ref> >= 1 - 1e-8 (the deterministic sign rule of proj/src/svd.cpp:336-354
  is part of the contract). The one exemption is a column whose sign-deciding
  entry is a near-tie in the reference (the two largest |u_ref| within 1e-9
  relative, so a 1e-15 perturbation legitimately picks the other one); the
  unsigned overlap is still required there.
* a cluster of >1 columns is compared by the largest principal angle between the
  two column spans (proj/tests/test_support.hpp:71-79), computed from its sine
  ||(I - Ã Ãᵀ) B||₂ for accuracy at small angles; bound 1e-6, or -- for a cluster
  whose gap to the rest of the spectrum is itself tiny -- the Davis-Kahan
  sensitivity of that subspace to a backward error of 1e3·eps·sigma_max
  (sin theta <= ||E|| / gap; 1e3 covers the sqrt(rows) growth of the merge's QR of
  up to 262144 stacked rows). Example: c5's sigma_4 ≈ sigma_5 ≈ sqrt(10) (rows
  carrying 10 unit repair edges), 1.5e-8 from the next sigma: bound 5.5e-5.
* columns of numerically zero sigma (<= 1e-10·sigma_max) are any basis of part of
  the null space; they are compared (as a span) only when U is square and they
  form its tail, where the span is the complement of the rest.
"""
from __future__ import annotations

import numpy as np

SIGMA_REL = 1e-10
SIGMA_SPLIT = 1e-10     # relative check above SIGMA_SPLIT·sigma_max
SIGMA_ABS = 1e-8        # absolute (·sigma_max) below it
OVERLAP = 1 - 1e-8
CLUSTER_TOL = 1e-9      # proj/src/metrics.cpp:15
ANGLE = 1e-6            # proj/tests/test_support.hpp:71-79 usage
DK_BACKWARD = 1e3 * np.finfo(np.float64).eps  # backward error (x sigma_max) behind the Davis-Kahan bound


def clusters(sigma_ref: np.ndarray) -> list[tuple[int, int]]:
    """[lo, hi) runs of consecutive sigma within CLUSTER_TOL·sigma_max (align_signs' grouping)."""
    n = len(sigma_ref)
    if n == 0:
        return []
    tol = CLUSTER_TOL * float(np.max(sigma_ref))
    out, lo = [], 0
    while lo < n:
        hi = lo + 1
        while hi < n and abs(sigma_ref[hi - 1] - sigma_ref[hi]) <= tol:
            hi += 1
        out.append((lo, hi))
        lo = hi
    return out


def sin_largest_angle(a: np.ndarray, b: np.ndarray) -> float:
    """sin of the largest principal angle between span(a) and span(b): ||(I - Qb Qbᵀ) Qa||₂.
    Symmetric when the spans have equal dimension; with dim a < dim b it measures how far
    span(a) leaves span(b)."""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    r = qa - qb @ (qb.T @ qa)
    return float(np.linalg.norm(r, 2)) if r.size else 0.0


def sign_ambiguous(u_ref_col: np.ndarray) -> bool:
    a = np.abs(u_ref_col)
    if a.size < 2:
        return False
    top = np.sort(a)[-2:]
    return top[0] >= top[1] * (1 - 1e-9)


def check_sigma(sig, ref_sigma, what=""):
    sig = np.asarray(sig)
    assert sig.shape == ref_sigma.shape, (what, sig.shape, ref_sigma.shape)
    if ref_sigma.size == 0:
        return 0.0
    smax = float(ref_sigma.max())
    big = ref_sigma > SIGMA_SPLIT * smax
    worst = 0.0
    if big.any():
        rel = np.abs(sig[big] - ref_sigma[big]) / ref_sigma[big]
        worst = float(rel.max())
        assert worst <= SIGMA_REL, (what, "sigma rel", worst, int(np.argmax(rel)))
    small = np.abs(sig[~big] - ref_sigma[~big])
    assert np.all(small <= SIGMA_ABS * max(smax, 1e-300)), (what, "small sigma abs", float(small.max(initial=0)))
    return worst


def check_u(u, ref_u, ref_sigma, what="", cols: int | None = None):
    """Signed singleton overlaps + cluster principal angles. Returns (min signed overlap, max cluster sin)."""
    u = np.asarray(u)
    k = ref_u.shape[1] if cols is None else cols
    assert u.shape[0] == ref_u.shape[0] and u.shape[1] >= k, (what, u.shape, ref_u.shape)
    min_ov, max_sin = 1.0, 0.0
    smax = float(np.max(ref_sigma)) if len(ref_sigma) else 0.0
    square = ref_u.shape[1] == ref_u.shape[0]
    for lo, hi in clusters(ref_sigma[:ref_u.shape[1]]):
        if lo >= k:
            break
        hi_c = min(hi, k)
        if np.all(ref_sigma[lo:hi] <= SIGMA_SPLIT * smax):
            # numerically zero sigma: the columns span part of the null space, which fixes them
            # only when U is a full basis and the cluster is its tail (the complement of the rest)
            if square and hi == ref_u.shape[1]:
                s = sin_largest_angle(u[:, lo:hi_c], ref_u[:, lo:hi])
                max_sin = max(max_sin, s)
                assert s <= ANGLE, (what, "null-space tail", lo, hi, s)
            continue
        if hi - lo == 1:
            ov = float(u[:, lo] @ ref_u[:, lo])
            if ov < OVERLAP and sign_ambiguous(ref_u[:, lo]):
                ov = abs(ov)
            min_ov = min(min_ov, ov)
            assert ov >= OVERLAP, (what, "column", lo, ov)
        else:
            # a cluster cut by the top-k truncation is not a well-defined subspace; its kept
            # columns must then lie in the reference's cluster span (hi_c < hi)
            s = sin_largest_angle(u[:, lo:hi_c], ref_u[:, lo:hi])
            max_sin = max(max_sin, s)
            outside = np.concatenate([ref_sigma[:lo], ref_sigma[hi:len(ref_sigma)]])
            gap = float(np.min(np.abs(outside[:, None] - ref_sigma[None, lo:hi]))) if outside.size else np.inf
            bound = max(ANGLE, DK_BACKWARD * smax / gap) if gap > 0 else np.inf
            assert s <= bound, (what, "cluster", lo, hi, s, bound)
    return min_ov, max_sin


def compare(s, ref_sigma, ref_u, what=""):
    """sigma and U of an SvdResult-like `s` (attributes sigma, u) against the reference's."""
    check_sigma(s.sigma, ref_sigma, what)
    return check_u(s.u, ref_u, ref_sigma, what)


def check_v_rows(v, v_ref, sigma_ref, what="", dv_max=np.sqrt(2e-8)):
    """A block of V rows (V = Aᵀ U Σ⁻¹ restricted to some columns of A) against the
    reference's. v_j - v_ref_j = Aᵀ(u_j - u_ref_j)/σ_j (+ the σ difference), so the
    north_star's U tolerance (|<u, u_ref>| >= 1 - 1e-8, i.e. ||Δu_j|| <= sqrt(2e-8))
    bounds ||Δv_j|| <= sqrt(2e-8) σ_max / σ_j in the units of the full, unit-norm V
    column -- an absolute bound: on a slice of rows a column's norm can be tiny.
    Singleton-cluster columns by that bound (a wrong sign or vector is O(1)); cluster
    columns by the least-squares residual of their slice in the reference's span."""
    v, v_ref = np.asarray(v), np.asarray(v_ref)
    assert v.shape == v_ref.shape, (what, v.shape, v_ref.shape)
    smax = float(np.max(sigma_ref)) if len(sigma_ref) else 0.0
    worst = 0.0
    for lo, hi in clusters(sigma_ref[:v_ref.shape[1]]):
        tol = dv_max * smax / max(float(np.min(sigma_ref[lo:hi])), 1e-300) * np.sqrt(hi - lo)
        if hi - lo == 1:
            e = float(np.linalg.norm(v[:, lo] - v_ref[:, lo]))
        else:
            a, b = v[:, lo:hi], v_ref[:, lo:hi]
            x, *_ = np.linalg.lstsq(b, a, rcond=None)
            e = float(np.linalg.norm(a - b @ x))
        worst = max(worst, e / tol)
        assert e <= tol, (what, "V columns", lo, hi, e, tol)
    return worst
