"""GPU run_pipeline (+ V) against the reference: the acceptance criteria
(proj/tests/acceptance_main.cpp) and the BASELINE configs c1/c2 end to end."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from parity import compare, check_u

pytestmark = pytest.mark.gpu


def sigma_error(a, b):
    """metrics.cpp:32-42"""
    n = max(len(a), len(b))
    a = np.pad(np.asarray(a, float), (0, n - len(a)))
    b = np.pad(np.asarray(b, float), (0, n - len(b)))
    return float(np.abs(a - b).sum())


def test_proxy_equivalence():
    # acceptance 1: dense 16x256, D in {2,4,8}, method none
    rng = np.random.default_rng(0)
    for seed in range(20):
        dense = rng.uniform(-1, 1, (16, 256))
        a = rk.sparse_of(dense)
        o = rk.dense_svd(dense)
        for d in (2, 4, 8):
            res = rk.run_pipeline(a, d, "none", 0, seed, 1)
            rel = np.abs(res.svd.sigma - o.sigma) / o.sigma
            assert rel.max() <= 1e-10
            assert float(res.svd.u[:, 0] @ o.u[:, 0]) >= 1 - 1e-8  # signed: the sign rule is shared


def repair_demo_instance():
    # acceptance_main.cpp:85-99 structure (8x64, row 7 lonely in block 0)
    rng = np.random.default_rng(123)
    e = []
    for r in range(7):
        for c in range(64):
            if rng.uniform() < 0.6:
                e.append((r, c, 1.0 + rng.uniform()))
    e += [(7, 40, 1.5), (7, 50, 2.0), (7, 63, 1.25)]
    return rk.SparseMatrix(8, 64, e)


def test_repair_necessity():
    # acceptance 2
    a = repair_demo_instance()
    none = rk.run_pipeline(a, 2, "none", 0, 0, 1)
    for m in ("random", "neighbor", "neighbor-random"):
        for seed in range(3):
            res = rk.run_pipeline(a, 2, m, 0, seed, 1)
            assert res.report.added_edges
            o = rk.dense_svd(res.repaired.to_dense())
            assert sigma_error(res.svd.sigma, o.sigma) <= 1e-9
            assert sigma_error(none.svd.sigma, o.sigma) > 1e-3


def test_table_regime(ref):
    # acceptance 3 (seeds 0-3 of 0-9), against the reference pipeline
    for seed in range(4):
        a = configs.synth_bipartite(64, 8192, 0.002, seed)
        r, c, v = a.coo()
        for d in (2, 8, 32):
            for m in ("random", "neighbor", "neighbor-random"):
                res = rk.run_pipeline(a, d, m, 0, seed, 1)
                o = ref.run_pipeline((64, 8192, r, c, v), d, m, 0, seed)
                assert np.array_equal(res.report.edges_array(), o.edges)
                assert sigma_error(res.svd.sigma, o.sigma) <= 1e-9
                compare(res.svd, o.sigma, o.u, f"seed {seed} D {d} {m}")


def test_determinism_and_workers():
    # acceptance 6: bitwise identical for any workers value and repeated runs
    for config in range(8):
        rows, cols = 4 + (config % 5) * 3, 32 + (config % 4) * 24
        a = configs.synth_bipartite(rows, cols, 0.04 + 0.03 * (config % 3), config)
        method = ["random", "neighbor", "neighbor-random", "none"][config % 4]
        keep = 3 if config % 6 == 5 else 0
        blocks = 1 + config % 8
        base = rk.run_pipeline(a, blocks, method, keep, config, 1)
        for workers in (4, 8):
            res = rk.run_pipeline(a, blocks, method, keep, config, workers)
            assert np.array_equal(res.svd.sigma, base.svd.sigma) and np.array_equal(res.svd.u, base.svd.u)
            assert all(x == y for x, y in zip(res.records, base.records))
            assert res.report.to_log() == base.report.to_log() and res.repaired == base.repaired


def test_single_block_equals_dense():
    # harness_test.cpp:146-156
    rng = np.random.default_rng(123)
    dense = rng.uniform(-1, 1, (5, 9))
    res = rk.run_pipeline(rk.sparse_of(dense), 1, "none", 0, 0, 1)
    o = rk.dense_svd(dense)
    assert np.max(np.abs(res.svd.sigma - o.sigma)) <= 1e-12 * o.sigma[0]


def test_pipeline_errors():
    # harness_test.cpp:174-194
    a = configs.synth_bipartite(4, 16, 0.5, 0)
    with pytest.raises(rk.InvalidArgument):
        rk.run_pipeline(a, 0, "none", 0, 0, 1)
    with pytest.raises(rk.InvalidArgument):
        rk.run_pipeline(a, 17, "none", 0, 0, 1)
    with pytest.raises(rk.InvalidArgument):
        rk.run_pipeline(a, 2, "none", 0, 0, 0)
    bad = rk.SparseMatrix(2, 8, [(0, 0, 1.0), (0, 5, np.inf), (1, 2, 1.0), (1, 7, 1.0)])
    with pytest.raises(rk.RankyRuntimeError, match="block task 1"):
        rk.run_pipeline(bad, 2, "none", 0, 0, 1)


def test_pipeline_records_shape():
    # harness_test.cpp:196-208
    a = configs.synth_bipartite(8, 64, 0.03, 10)
    res = rk.run_pipeline(a, 8, "neighbor", 0, 2, 2)
    for d in range(8):
        assert rk.find_lonely_rows(res.repaired, res.partition, d) == []
        assert res.records[d].block_index == d and res.records[d].rows == 8 and res.records[d].kept == 8


def test_reference_fixture_pipelines(golden, garrays):
    for name, p in golden["pipelines"].items():
        shape = garrays[f"pipe_{name}_shape"]
        a = rk.SparseMatrix._trusted(int(shape[0]), int(shape[1]), rk.ranky._entries(
            garrays[f"pipe_{name}_r"], garrays[f"pipe_{name}_c"], garrays[f"pipe_{name}_v"]))
        res = rk.run_pipeline(a, p["D"], p["method"], p["keep"], p["seed"], 1, want_v=True)
        assert np.array_equal(res.report.edges_array(), garrays[f"pipe_{name}_edges"])
        compare(res.svd, garrays[f"pipe_{name}_sigma"], garrays[f"pipe_{name}_u"], name)
        for d in range(p["records"]):
            # a record is U*Sigma of one block: its column norms are the block's
            # singular values and P P^T = A_d A_d^T is independent of the basis
            # chosen inside degenerate clusters (value-1.0 blocks have many)
            want = garrays[f"pipe_{name}_rec{d}"]
            got = res.records[d].payload.reshape(want.shape)
            scale = max(1.0, float(np.abs(want).max())) ** 2
            assert np.allclose(np.linalg.norm(got, axis=0), np.linalg.norm(want, axis=0), rtol=1e-10,
                               atol=1e-12 * scale), (name, d)
            assert np.max(np.abs(got @ got.T - want @ want.T)) <= 1e-12 * scale * want.shape[0], (name, d)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_baseline_config_end_to_end(name, ref):
    cfg = configs.CONFIGS[name]
    a = cfg.generate()
    r, c, v = a.coo()
    res = rk.run_pipeline(a, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True, top_k=cfg.top_k)
    o = ref.full_svd((a.rows(), a.cols(), r, c, v), cfg.blocks, cfg.method, cfg.keep, cfg.seed, 8, cfg.top_k) \
        if ref.kind == "reference" else None
    if o is None:
        o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), cfg.blocks, cfg.method, cfg.keep, cfg.seed)
        o.v = ref.recover_right_vectors(o.matrix, o.u, o.sigma, 1e-10)
    compare(res.svd, o.sigma, o.u, name)
    # V against the reference's own V: signed per column, clusters by principal angle
    assert res.svd.v.shape == o.v.shape
    check_u(res.svd.v, o.v, o.sigma[:o.v.shape[1]], f"{name} V")
    # bit-exact V given identical U, sigma and repaired matrix
    vr = ref.recover_right_vectors((a.rows(), a.cols(), *res.repaired.coo()), res.svd.u, res.svd.sigma, 1e-10)
    assert np.array_equal(res.svd.v, vr)


@pytest.mark.parametrize("route", ["auto", "householder"])
def test_block_routes_agree(route, tuning_env, ref):
    """The Gram/Cholesky route (accepted only when kappa <= kappa_max(M)) and the
    Householder route both reproduce the reference on c1 (ill-conditioned blocks:
    mostly Householder) and a c2 slice (well-conditioned: Gram)."""
    tuning_env("RK_BLOCK_ROUTE", route)
    for name, scale in (("c1", None), ("c2", 262144 // 8)):
        cfg = configs.CONFIGS[name]
        a = cfg.generate(scale)
        r, c, v = a.coo()
        blocks = cfg.blocks if scale is None else cfg.blocks // 8
        res = rk.run_pipeline(a, blocks, cfg.method, cfg.keep, cfg.seed, 1)
        o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), blocks, cfg.method, cfg.keep, cfg.seed)
        compare(res.svd, o.sigma, o.u, f"{name} {route}")


@pytest.mark.parametrize("env", [("RK_PRECOND", "1"), ("RK_CHOL", "r"), ("RK_SPMM_WARP", "1"), ("RK_DIAG_ORDER", "0")])
def test_variant_switches_agree(env, tuning_env, ref):
    """The opt-in variants (FP32-preconditioned Jacobi, the right-looking Cholesky,
    the one-warp-per-column V SpMM, the Gram route without diagonal ordering)
    reproduce the reference on a c2 slice like the defaults: only how the result
    is reached changes, not the stopping rule or the V arithmetic."""
    if env[0] in ("RK_PRECOND", "RK_CHOL") and not rk.ranky.experiments_built():
        pytest.skip("measured-and-not-kept variant: experiments build only (RK_EXPERIMENTS=1)")
    tuning_env(*env)
    cfg = configs.CONFIGS["c2"]
    scale = 262144 // 8
    a = cfg.generate(scale)
    r, c, v = a.coo()
    blocks = cfg.blocks // 8
    res = rk.run_pipeline(a, blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
    o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), blocks, cfg.method, cfg.keep, cfg.seed)
    compare(res.svd, o.sigma, o.u, f"c2 slice {env}")
    vr = ref.recover_right_vectors((a.rows(), a.cols(), *res.repaired.coo()), res.svd.u, res.svd.sigma, 1e-10)
    assert np.array_equal(res.svd.v, vr)


@pytest.mark.parametrize("env", [("RK_JACOBI_SMEM", "0"), ("RK_JACOBI_SMEM_CL", "1"), ("RK_JACOBI_CARRY", "0"),
                                 ("RK_APPLY_Q", "panel"), ("RK_PRESENCE", "csr")])
def test_wide_block_variants_agree(env, tuning_env, ref):
    """c3's route (wide blocks: QR of X = T^T, Jacobi on R, apply_q; NeighborChecker) against the
    reference's run_pipeline on a 16-block slice, with the round-2 kernels switched off one at a
    time: the direct Jacobi instead of the shared-memory Gram-assisted one, one-CTA jobs only (the
    larger R factors then take the direct kernel), the full 16 x 16 Gram every step instead of carried
    diagonal blocks, apply_q reflector by reflector instead of
    compact-WY, the rank check from the CSR instead of the CSC slices."""
    tuning_env(*env)
    cfg = configs.CONFIGS["c3"]
    blocks = 16
    a = cfg.generate(8192 * blocks)
    r, c, v = a.coo()
    res = rk.run_pipeline(a, blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
    o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), blocks, cfg.method, cfg.keep, cfg.seed)
    assert np.array_equal(res.report.edges_array(), o.edges)
    compare(res.svd, o.sigma, o.u, f"c3 slice {env}")
    vr = ref.recover_right_vectors((a.rows(), a.cols(), *res.repaired.coo()), res.svd.u, res.svd.sigma, 1e-10)
    assert np.array_equal(res.svd.v, vr)


def test_syrk_block_kernel_bitwise(tuning_env):
    """The merge's SYRK with a 32 x 32 block per warp (default) and with one 8 x 8 tile per warp
    (RK_SYRK=tile) accumulate every tile's k-steps in the same order: the pipeline's outputs are
    bitwise the same."""
    cfg = configs.CONFIGS["c2"]
    a = cfg.generate(262144 // 4)
    outs = []
    for mode in ("block", "tile"):
        tuning_env("RK_SYRK", mode)
        res = rk.run_pipeline(a, cfg.blocks // 4, cfg.method, cfg.keep, cfg.seed, 1)
        outs.append((res.svd.sigma.copy(), res.svd.u.copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_gram_kernels_bitwise(tuning_env):
    """The block Gram from rows x columns (default) and from row pairs (the
    merge-join kernel, RK_GRAM_PAIRS=1) add every G(r, s) in ascending column
    order from zero: the pipeline's outputs are bitwise the same."""
    from paper_2009_09767_b200 import ranky as R
    if not R.experiments_built():
        pytest.skip("the row-pair Gram kernel is in the experiments build only (RK_EXPERIMENTS=1)")
    cfg = configs.CONFIGS["c2"]
    a = cfg.generate(262144 // 4)
    dm = rk.DeviceMatrix(a)
    outs = []
    for flag in ("0", "1"):
        tuning_env("RK_GRAM_PAIRS", flag)
        out, _ = R.dev_full_svd(dm, cfg.blocks // 4, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
        sig, u, v = R.dev_outputs_tensors(out)
        outs.append((sig.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()))
        R.dev_outputs_free(out)
    for x, y in zip(outs[0], outs[1]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("eig", ["1", "0"])
def test_merge_gram_routes_agree(eig, tuning_env, ref):
    """The merge's Gram route by the symmetric eigensolver (tridiagonalisation in one
    cluster, bisection, inverse iteration; rk_eig.cu) and by Cholesky + one-sided
    Jacobi (RK_EIG_MERGE=0) both reproduce the reference's run_pipeline on c2 slices
    (well-conditioned merges: the Gram route is taken) and on c1 (rejected: TSQR)."""
    tuning_env("RK_EIG_MERGE", eig)
    cfg = configs.CONFIGS["c2"]
    for scale, blocks in ((262144 // 8, 8), (262144 // 4, 16), (262144 // 16, 4)):
        a = cfg.generate(scale)
        r, c, v = a.coo()
        res = rk.run_pipeline(a, blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True)
        o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), blocks, cfg.method, cfg.keep, cfg.seed)
        compare(res.svd, o.sigma, o.u, f"c2 slice {scale} eig {eig}")
    c1 = configs.CONFIGS["c1"]
    a = c1.generate()
    r, c, v = a.coo()
    res = rk.run_pipeline(a, c1.blocks, c1.method, c1.keep, c1.seed, 1)
    o = ref.run_pipeline((a.rows(), a.cols(), r, c, v), c1.blocks, c1.method, c1.keep, c1.seed)
    compare(res.svd, o.sigma, o.u, f"c1 eig {eig}")
