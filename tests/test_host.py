"""Host-side logic of the Python mirror (containers, argument checks, formats)
and the workload generators. CPU only; mirrors proj/tests/sparse_core_test.cpp,
harness_test.cpp and parts of repair_test.cpp."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200.ranky import (AddedEdge, RepairMethod, RepairReport, rank_equal_probability,
                                         repair_method_from_string, to_string)


def test_sparse_matrix_validation():
    a = rk.SparseMatrix(3, 4, [(2, 1, 1.0), (0, 3, 2.0), (0, 1, -1.0)])
    assert a.nnz() == 3
    assert [tuple(e) for e in a.entries()] == [(0, 1, -1.0), (0, 3, 2.0), (2, 1, 1.0)]
    assert a.count_in_columns(0, 0, 2) == 1
    with pytest.raises(rk.InvalidArgument, match="outside"):
        rk.SparseMatrix(2, 2, [(2, 0, 1.0)])
    with pytest.raises(rk.InvalidArgument, match="stores zero"):
        rk.SparseMatrix(2, 2, [(0, 0, 0.0)])
    with pytest.raises(rk.InvalidArgument, match="duplicate"):
        rk.SparseMatrix(2, 2, [(0, 0, 1.0), (0, 0, 2.0)])
    with pytest.raises(rk.OutOfRange):
        a.row_entries(5)
    # the first violating entry in sorted order decides (sparse_matrix.cpp:15-29): an early
    # stored zero is reported before a later out-of-range entry, and vice versa
    with pytest.raises(rk.InvalidArgument, match=r"\(0, 1\) stores zero"):
        rk.SparseMatrix(2, 2, [(5, 0, 1.0), (0, 1, 0.0)])
    with pytest.raises(rk.InvalidArgument, match=r"\(0, 7\) outside"):
        rk.SparseMatrix(2, 2, [(0, 7, 1.0), (1, 1, 0.0)])
    with pytest.raises(rk.InvalidArgument, match=r"duplicate sparse entry \(0, 1\)"):
        rk.SparseMatrix(2, 2, [(1, 1, 0.0), (0, 1, 2.0), (0, 1, 3.0)])


def test_partition_columns():
    # proj/src/partition.cpp:38-51: remainder goes to the last block
    p = rk.partition_columns(10, 3)
    assert [(r.begin, r.end) for r in p.ranges()] == [(0, 3), (3, 6), (6, 10)]
    assert p.block_of(9) == 2 and p.block_of(3) == 1
    with pytest.raises(rk.InvalidArgument):
        rk.partition_columns(4, 0)
    with pytest.raises(rk.InvalidArgument):
        rk.partition_columns(4, 5)
    with pytest.raises(rk.OutOfRange):
        p.range(3)
    for n in range(1, 40):
        for d in range(1, n + 1):
            q = rk.partition_columns(n, d)
            assert q.ranges()[-1].end == n and all(r.width() >= 1 for r in q.ranges())


def test_block_view():
    a = rk.SparseMatrix(2, 6, [(0, 0, 1.0), (0, 4, 2.0), (1, 5, 3.0)])
    b = rk.block_view(a, rk.partition_columns(6, 2), 1)
    assert b.cols() == 3 and [tuple(e) for e in b.entries()] == [(0, 1, 2.0), (1, 2, 3.0)]


def test_report_log_and_names():
    rep = RepairReport([AddedEdge(0, 1, 0, RepairMethod.kNeighbor)], [1, 0], 0)
    assert rep.to_log() == "0\t1\t0\tneighbor\n# lonely=1,0 fallback=0\n"
    for m in RepairMethod:
        assert repair_method_from_string(to_string(m)) == m
    with pytest.raises(rk.InvalidArgument):
        repair_method_from_string("ransom")


def test_rank_equal_probability():
    # proj/tests/repair_test.cpp:287-294
    assert rank_equal_probability(500, 3) == 0.994
    assert rank_equal_probability(100, 0) == 1.0
    assert rank_equal_probability(100, 150) == 0.0
    with pytest.raises(rk.InvalidArgument):
        rank_equal_probability(0, 3)


def test_proxy_from_records_order_and_errors():
    recs = [rk.BlockResultRecord(1, 2, 1, np.array([3.0, 4.0])), rk.BlockResultRecord(0, 2, 2, np.arange(4.0))]
    p = rk.proxy_from_records(recs, 2)
    assert p.block_offsets == [0, 2, 3]
    assert np.array_equal(p.matrix, np.array([[0.0, 1.0, 3.0], [2.0, 3.0, 4.0]]))
    with pytest.raises(rk.InvalidArgument, match="duplicate"):
        rk.proxy_from_records(recs + [recs[0]], 2)
    with pytest.raises(rk.InvalidArgument, match="rows"):
        rk.proxy_from_records(recs, 3)


def test_build_proxy():
    res = [rk.SvdResult(np.eye(2), np.array([2.0, 1.0])), rk.SvdResult(np.ones((2, 1)), np.array([0.5]))]
    p = rk.build_proxy(res, 2)
    assert p.block_offsets == [0, 2, 3] and p.matrix[0, 0] == 2.0 and p.matrix[1, 2] == 0.5
    with pytest.raises(rk.InvalidArgument):
        rk.build_proxy(res, 3)


def test_generators_are_deterministic_and_match_spec():
    c1 = configs.CONFIGS["c1"]
    a, b = c1.generate(), c1.generate()
    assert a == b
    e = a.entries()
    assert a.rows() == 64 and a.cols() == 8192
    assert 0.008 < a.nnz() / (64 * 8192) < 0.011
    assert np.all(np.abs(e["value"]) < 1) and np.all(e["value"] != 0)
    # 8 rows emptied inside 4 blocks (BASELINE configs[0])
    p = rk.partition_columns(8192, 16)
    empty = 0
    for d in range(16):
        rg = p.range(d)
        rows_with = set(e["row"][(e["col"] >= rg.begin) & (e["col"] < rg.end)].tolist())
        empty += sum(1 for r in range(64) if r not in rows_with)
    assert empty >= 32
    s = configs.synth_bipartite(64, 8192, 0.002, 7)
    assert s.nnz() == 1025  # proj/tests/sparse_core_test.cpp:21


def test_c2_shape_and_planted_rows():
    a = configs.CONFIGS["c2"].generate()
    assert a.rows() == 256 and a.cols() == 262144
    assert 0.0045 < a.nnz() / (256 * 262144) < 0.0055
    e = a.entries()
    v = e["value"]
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01  # N(0,1)


def test_planted_generator_spectrum():
    """c5 generator: with a full mask and no noise A = P diag(0.9^k) Q^T exactly,
    so its singular values are 0.9^k (k < 64) and ~0 after; deterministic; the
    mask density and the noise level follow the spec."""
    a = configs.planted(128, 4096, 1.0, 64, 0.9, 0.0, 7)
    assert a.nnz() == 128 * 4096
    s = np.linalg.svd(a.to_dense(), compute_uv=False)
    assert np.abs(s[:64] - 0.9 ** np.arange(64)).max() < 1e-13
    assert s[64] < 1e-13
    b = configs.planted(256, 65536, 0.0005, 64, 0.9, 1e-6, 4)
    assert np.array_equal(b.entries(), configs.planted(256, 65536, 0.0005, 64, 0.9, 1e-6, 4).entries())
    assert abs(b.nnz() / (256 * 65536) - 0.0005) < 0.00005
    r, c, v = b.coo()
    assert np.all(v != 0) and np.all(np.diff(r.astype(np.int64)) >= 0)
    # the noise is additive on the same mask: the difference of two noise levels is noise
    z0 = configs.planted(64, 8192, 0.01, 64, 0.9, 0.0, 3)
    z1 = configs.planted(64, 8192, 0.01, 64, 0.9, 1e-6, 3)
    assert np.array_equal(z0.coo()[1], z1.coo()[1])
    assert 0.5e-6 < np.std(z1.coo()[2] - z0.coo()[2]) < 2e-6


def test_keyed_rng_host_object_kat():
    # KeyedRng(0,0,0)'s first draws as the reference library produces them (SURVEY.md §8(c)
    # lists the same three values, last first); repair_test.cpp:77-88
    from paper_2009_09767_b200.ranky import KeyedRng
    g = KeyedRng(0, 0, 0)
    assert [g.next() for _ in range(3)] == [0x060599146f06297d, 0x0bc1da82f6532f86, 0x9cd8ff1831b74722]
    assert 0 <= KeyedRng(42, 0, 8).below(1024) < 1024
    u = KeyedRng(1, 2, 3).unit()
    assert 0.0 <= u < 1.0
