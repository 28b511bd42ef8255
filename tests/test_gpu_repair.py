"""GPU rank check + checker repair: bit-exact against the reference
(fixtures from the unmodified reference, and the live CPU oracle).
Mirrors proj/tests/repair_test.cpp."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from conftest import golden_matrix

pytestmark = pytest.mark.gpu


def sm(rows, cols, entries):
    return rk.SparseMatrix(rows, cols, entries)


def test_keyed_rng_on_device(golden):
    for case in golden["rng"]:
        s, b, r = case["key"]
        out = rk.keyed_rng_next(s, [b], [r], 5)[0]
        assert [str(int(x)) for x in out] == case["next"]
    for case in golden["rng_below"]:
        s, b, r = case["key"]
        assert int(rk.keyed_rng_below(s, [b], [r], [case["bound"]])[0]) == case["value"]


def test_random_checker_regression():
    # repair_test.cpp:77-88: first lonely row of block 0 at D=8 is 8; seed 42 picks column 587
    a = configs.synth_bipartite(64, 8192, 0.002, 7)
    p = rk.partition_columns(8192, 8)
    lonely = rk.find_lonely_rows(a, p, 0)
    assert lonely and lonely[0] == 8
    assert int(rk.keyed_rng_below(42, [0], [8], [1024])[0]) == 587
    rep, report = rk.repair(a, p, "random", 42)
    first = [e for e in report.added_edges if e.block == 0][0]
    assert (first.row, first.col) == (8, 587)


def test_repair_fixtures_bit_exact(golden, garrays):
    for name, case in golden["repair"].items():
        r, c, v = golden_matrix(garrays, name)
        a = rk.SparseMatrix._trusted(case["rows"], case["cols"], rk.ranky._entries(r, c, v))
        repaired, report = rk.repair(a, rk.partition_columns(case["cols"], case["D"]), case["method"], case["seed"])
        assert report.edges_array().tolist() == case["edges"], name
        assert report.lonely_counts == case["lonely"], name
        assert report.fallback_count == case["fallback"], name
        assert report.to_log() == case["log"], name
        assert repaired.nnz() == case["repaired_nnz"], name


def test_repair_against_live_oracle(ref):
    for seed in range(4):
        for (m, n, dens, D) in [(8, 16, 0.12, 4), (12, 96, 0.015, 6), (32, 2000, 0.01, 20), (64, 8192, 0.003, 64)]:
            a = configs.synth_bipartite(m, n, dens, seed)
            r, c, v = a.coo()
            for meth in ("random", "neighbor", "neighbor-random", "none"):
                repaired, report = rk.repair(a, rk.partition_columns(n, D), meth, 11 * seed + 1)
                o = ref.repair((m, n, r, c, v), D, meth, 11 * seed + 1)
                assert np.array_equal(report.edges_array().reshape(-1, 4), o.edges.reshape(-1, 4)), (seed, m, meth)
                assert report.lonely_counts == o.lonely_counts.tolist()
                assert report.fallback_count == o.fallback_count
                rr, rc, rv = repaired.coo()
                assert np.array_equal(rr, o.matrix[2]) and np.array_equal(rc, o.matrix[3])
                assert np.array_equal(rv, o.matrix[4])


def test_c1_and_c2_repair_bit_exact(ref):
    for name in ("c1", "c2"):
        cfg = configs.CONFIGS[name]
        a = cfg.generate()
        r, c, v = a.coo()
        for meth in ("random", "neighbor", "neighbor-random"):
            repaired, report = rk.repair(a, rk.partition_columns(a.cols(), cfg.blocks), meth, cfg.seed)
            o = ref.repair((a.rows(), a.cols(), r, c, v), cfg.blocks, meth, cfg.seed)
            assert np.array_equal(report.edges_array(), o.edges), (name, meth)
            assert report.lonely_counts == o.lonely_counts.tolist()
            assert report.fallback_count == o.fallback_count


def test_neighbor_semantics():
    # repair_test.cpp:90-102: the only eligible columns are row 0's block-0 entries
    a = sm(3, 6, [(0, 0, 1.0), (0, 2, 1.0), (0, 5, 1.0), (1, 5, 1.0), (2, 1, 1.0)])
    _, report = rk.repair(a, rk.partition_columns(6, 2), "neighbor", 3)
    e = [x for x in report.added_edges if x.block == 0 and x.row == 1][0]
    assert e.col in (0, 2) and e.mechanism == rk.RepairMethod.kNeighbor


def test_isolated_row_fallback():
    # repair_test.cpp:264-273
    a = sm(3, 6, [(0, 0, 1.0), (2, 1, 1.0)])
    p = rk.partition_columns(6, 1)
    repaired, report = rk.repair(a, p, "neighbor", 0)
    assert report.fallback_count == 1 and len(report.added_edges) == 1
    assert report.added_edges[0].mechanism == rk.RepairMethod.kRandom
    assert rk.find_lonely_rows(repaired, p, 0) == []


def test_empty_and_dense():
    # repair_test.cpp:175-195
    a = sm(3, 6, [])
    p = rk.partition_columns(6, 2)
    repaired, report = rk.repair(a, p, "random", 9)
    assert len(report.added_edges) == 6 and repaired.nnz() == 6 and report.lonely_counts == [3, 3]
    d = configs.synth_bipartite(4, 8, 1.0, 1)
    for m in ("random", "neighbor", "neighbor-random", "none"):
        rep, report = rk.repair(d, rk.partition_columns(8, 4), m, 5)
        assert rep == d and not report.added_edges and report.fallback_count == 0


def test_postconditions():
    # repair_test.cpp:218-243
    a = configs.synth_bipartite(12, 96, 0.015, 21)
    p = rk.partition_columns(96, 6)
    for m in ("random", "neighbor", "neighbor-random"):
        repaired, report = rk.repair(a, p, m, 4)
        for d in range(6):
            assert rk.find_lonely_rows(repaired, p, d) == []
            assert report.lonely_counts[d] == len(rk.find_lonely_rows(a, p, d))
        for e in report.added_edges:
            rg = p.range(e.block)
            assert rg.begin <= e.col < rg.end
            assert a.count_in_columns(e.row, rg.begin, rg.end) == 0
            vals = [x["value"] for x in repaired.row_entries(e.row) if x["col"] == e.col]
            assert vals == [1.0]
        assert repaired.nnz() == a.nnz() + len(report.added_edges)


def test_planted_neighbor_workload(ref):
    """NeighborChecker / NeighborRandom on a c3-like Zipf matrix with planted empty
    rows (the ordered replay with many interacting lonely rows)."""
    base = configs.zipf(128, 40960, 0.256, 1.1, configs.VAL_UNIFORM_01, 5)
    e = base.entries()
    keep = ~((e["row"] % 7 == 3) & ((e["col"] // 1024) % 3 == 1))
    a = rk.SparseMatrix._trusted(128, 40960, e[keep].copy())
    r, c, v = a.coo()
    for meth in ("neighbor", "neighbor-random"):
        repaired, report = rk.repair(a, rk.partition_columns(40960, 40), meth, 2)
        o = ref.repair((128, 40960, r, c, v), 40, meth, 2)
        assert sum(report.lonely_counts) > 100
        assert np.array_equal(report.edges_array(), o.edges), meth
        assert report.fallback_count == o.fallback_count


def test_bad_arguments():
    a = configs.synth_bipartite(4, 16, 0.5, 0)
    with pytest.raises(rk.InvalidArgument):
        rk.repair(a, rk.partition_columns(8, 2), "random", 0)
    with pytest.raises(rk.OutOfRange):
        rk.find_lonely_rows(a, rk.partition_columns(16, 2), 5)


@pytest.mark.parametrize("method", ["neighbor", "neighbor-random"])
def test_speculated_replay_is_exact(method, tuning_env, ref):
    """The neighbor replay with speculated sets (every step's candidate and neighbor
    sets from the input alone, recomputed only where an earlier edge could change
    them) gives the reference's edges bit for bit -- on dense-collision cases (many
    lonely rows per block, rows lonely in several blocks) as on sparse ones."""
    cases = [(configs.synth_bipartite(16, 256, 0.03, s), 16) for s in range(4)]
    cases += [(configs.synth_bipartite(64, 8192, 0.002, 7), 32), (configs.synth_bipartite(200, 4000, 0.004, 3), 40)]
    for spec in ("1", "0"):
        tuning_env("RK_REPAIR_SPECULATE", spec)
        for a, D in cases:
            p = rk.partition_columns(a.cols(), D)
            rep, report = rk.repair(a, p, method, 11)
            r, c, v = a.coo()
            o = ref.repair((a.rows(), a.cols(), r, c, v), D, method, 11)
            assert np.array_equal(report.edges_array(), o.edges), (spec, a.rows(), D)
            assert report.fallback_count == o.fallback_count
