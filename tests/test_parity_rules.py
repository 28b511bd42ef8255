"""The parity checker itself (tests/parity.py), on CPU: a sign flip, a wrong
cluster subspace and a 1e-9 relative sigma error must all be caught; a rotation
inside a degenerate cluster and a sign flip of a near-tie column must pass."""
import numpy as np
import pytest

from parity import check_sigma, check_u, clusters, compare


def _svd_pair(seed=0, m=12, n=12, sigma=None):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    s = np.sort(rng.uniform(1, 2, n))[::-1] if sigma is None else np.asarray(sigma, float)
    # the reference sign rule: first max |u_ij| positive (proj/src/svd.cpp:336-354)
    for j in range(n):
        i = int(np.argmax(np.abs(u[:, j])))
        if u[i, j] < 0:
            u[:, j] = -u[:, j]
    return u, s


class R:
    def __init__(self, sigma, u):
        self.sigma, self.u = sigma, u


def test_identical_passes():
    u, s = _svd_pair()
    assert compare(R(s, u), s, u)[0] >= 1 - 1e-15


def test_sign_flip_caught():
    u, s = _svd_pair()
    bad = u.copy()
    bad[:, 3] = -bad[:, 3]
    with pytest.raises(AssertionError):
        compare(R(s, bad), s, u)


def test_sigma_rel_caught():
    u, s = _svd_pair()
    bad = s.copy()
    bad[5] *= 1 + 1e-9
    with pytest.raises(AssertionError):
        check_sigma(bad, s)
    ok = s.copy()
    ok[5] *= 1 + 1e-11
    check_sigma(ok, s)


def test_cluster_rotation_passes_and_wrong_subspace_caught():
    sig = [5.0, 3.0, 3.0, 3.0, 1.0, 0.5]
    u, s = _svd_pair(1, 8, 6, sig)
    assert clusters(s) == [(0, 1), (1, 4), (4, 5), (5, 6)]
    c, sn = np.cos(0.7), np.sin(0.7)
    rot = u.copy()
    rot[:, 1], rot[:, 2] = c * u[:, 1] + sn * u[:, 2], -sn * u[:, 1] + c * u[:, 2]
    compare(R(s, rot), s, u)
    bad = u.copy()
    bad[:, 2] = np.cos(1e-4) * u[:, 2] + np.sin(1e-4) * u[:, 4]   # leaves the cluster span
    bad[:, 4] = -np.sin(1e-4) * u[:, 2] + np.cos(1e-4) * u[:, 4]
    with pytest.raises(AssertionError):
        check_u(bad, u, s)


def test_small_sigma_absolute():
    s = np.array([1.0, 0.5, 1e-12, 0.0])
    check_sigma(np.array([1.0, 0.5, 3e-12, 1e-11]), s)
    with pytest.raises(AssertionError):
        check_sigma(np.array([1.0, 0.5, 1e-12, 1e-7]), s)


def test_near_tie_sign_exempt():
    u = np.eye(4)
    u[:, 0] = np.array([1, -1, 0, 0]) / np.sqrt(2)   # |u_00| == |u_10|: the sign rule is a tie
    u[:, 1] = np.array([1, 1, 0, 0]) / np.sqrt(2)
    s = np.array([4.0, 3.0, 2.0, 1.0])
    flipped = u.copy()
    flipped[:, 0] *= -1
    check_u(flipped, u, s)


def test_null_space_columns():
    rng = np.random.default_rng(4)
    u, _ = np.linalg.qr(rng.standard_normal((9, 9)))
    s = np.array([5.0, 2.0] + [1e-16] * 7)
    other = u.copy()
    q, _ = np.linalg.qr(rng.standard_normal((7, 7)))
    other[:, 2:] = u[:, 2:] @ q          # another basis of the same null space: passes
    check_u(other, u, s)
    trunc_ref, trunc = u[:, :4], other[:, :4]   # truncated: the null columns are not determined
    check_u(trunc, trunc_ref, s[:4])
