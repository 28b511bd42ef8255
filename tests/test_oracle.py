"""The CPU oracle (oracle/ranky_oracle.c) pinned against the reference's own
golden values and against fixtures generated from the unmodified reference
(tests/golden/make_golden.py). CPU only."""
import numpy as np
import pytest

from conftest import golden_matrix


def test_rng_streams(port, golden):
    for case in golden["rng"]:
        s, b, r = case["key"]
        assert [str(x) for x in port.rng_stream(s, b, r, 5)] == case["next"]
    for case in golden["rng_below"]:
        s, b, r = case["key"]
        assert port.rng_below(s, b, r, case["bound"]) == case["value"]


def test_reference_test_goldens(port, golden):
    # proj/tests/sparse_core_test.cpp:21 (nnz 1025), repair_test.cpp:77-88 (row 8 -> column 587)
    g = golden["synth_64_8192_0.002_7"]
    a = port.synth_bipartite(64, 8192, 0.002, 7)
    assert len(a[2]) == g["nnz"] == 1025
    lonely = port.find_lonely_rows(a, 8, 0)
    assert list(lonely) == g["lonely_block0_D8"]
    assert lonely[0] == 8
    assert port.rng_below(42, 0, 8, 1024) == g["random_col_seed42_row8"] == 587


def test_repair_matches_reference_fixtures(port, golden, garrays):
    for name, case in golden["repair"].items():
        r, c, v = golden_matrix(garrays, name)
        res = port.repair((case["rows"], case["cols"], r, c, v), case["D"], case["method"], case["seed"])
        edges = res.edges.tolist() if res.edges is not None else []
        assert edges == case["edges"], name
        assert res.lonely_counts.tolist() == case["lonely"], name
        assert res.fallback_count == case["fallback"], name
        assert res.to_log() == case["log"], name


def test_repair_log_golden(port, golden):
    # proj/tests/repair_test.cpp:253-262
    log = golden["repair"]["log_format"]["log"]
    assert log.startswith("0\t1\t0\tneighbor\n")
    assert "# lonely=1,0 fallback=0\n" in log


def test_dense_svd_matches_reference_bitwise(port, garrays):
    names = sorted({k[len("dense_"):-len("_a")] for k in garrays.files if k.startswith("dense_") and k.endswith("_a")})
    assert names
    for n in names:
        a = garrays[f"dense_{n}_a"]
        s = port.dense_svd(a)
        # same algorithm, same operation order, no contraction: identical bits
        assert np.array_equal(s.sigma, garrays[f"dense_{n}_sigma"]), n
        assert np.array_equal(s.u, garrays[f"dense_{n}_u"]), n
        assert np.array_equal(s.v, garrays[f"dense_{n}_v"]), n


def test_closed_forms(port):
    # proj/tests/svd_test.cpp:37-67
    assert list(port.dense_svd(np.eye(2)).sigma) == [1.0, 1.0]
    s = port.dense_svd(np.diag([3.0, 2.0]))
    assert list(s.sigma) == [3.0, 2.0] and s.u[0, 0] == 1.0 and s.u[1, 1] == 1.0
    s = port.dense_svd(np.array([[0, 0, 0, 0], [6.0, 0, 0, 8.0]]))
    assert abs(s.sigma[0] - 10) <= 1e-12 and abs(s.sigma[1]) <= 1e-13


def test_block_svd_matches_reference(port, garrays):
    keys = sorted({k[:-len("_sigma")] for k in garrays.files if k.startswith("block_") and k.endswith("_sigma")})
    for key in keys:
        m, n = (int(x) for x in key.split("_")[1].split("x"))
        blk = (m, n, garrays[key + "_r"], garrays[key + "_c"], garrays[key + "_v"])
        s = port.block_svd(blk, m)
        assert np.array_equal(s.sigma, garrays[key + "_sigma"]), key
        assert np.array_equal(s.u, garrays[key + "_u"]), key


def test_pipeline_matches_reference(port, golden, garrays):
    for name, p in golden["pipelines"].items():
        shape = garrays[f"pipe_{name}_shape"]
        a = (int(shape[0]), int(shape[1]), garrays[f"pipe_{name}_r"], garrays[f"pipe_{name}_c"],
             garrays[f"pipe_{name}_v"])
        res = port.run_pipeline(a, p["D"], p["method"], p["keep"], p["seed"])
        assert np.array_equal(res.sigma, garrays[f"pipe_{name}_sigma"]), name
        assert np.array_equal(res.u, garrays[f"pipe_{name}_u"]), name
        for d in range(p["records"]):
            assert np.array_equal(res.records[d], garrays[f"pipe_{name}_rec{d}"]), (name, d)
        v = port.recover_right_vectors(res.matrix, res.u, res.sigma, 1e-10)
        assert np.array_equal(v, garrays[f"pipe_{name}_V"]), name


def test_errors(port):
    from oracle import OracleError
    with pytest.raises(OracleError) as e:
        port.dense_svd(np.array([[1.0, np.nan]]))
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        port.run_pipeline((2, 8, np.array([0, 0, 1, 1], np.uint64), np.array([0, 5, 2, 7], np.uint64),
                           np.array([1.0, np.inf, 1.0, 1.0])), 2, "none", 0, 0)
    assert "block task 1" in str(e.value)  # proj/tests/harness_test.cpp:184-194
    with pytest.raises(OracleError):
        port.run_pipeline((2, 8, np.array([0], np.uint64), np.array([0], np.uint64), np.array([1.0])), 9, "none")


def test_restatement_agrees_with_live_reference(ref, port):
    if ref.kind != "reference":
        pytest.skip("reference not built here")
    for seed in range(4):
        a = port.synth_bipartite(24, 300, 0.04, seed)
        for m in ("random", "neighbor", "neighbor-random"):
            x, y = port.run_pipeline(a, 5, m, 0, seed), ref.run_pipeline(a, 5, m, 0, seed, 3)
            assert np.array_equal(x.edges, y.edges)
            assert np.array_equal(x.sigma, y.sigma) and np.array_equal(x.u, y.u)
