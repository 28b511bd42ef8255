"""Matrix Market through the C ABI (rk_load_matrix_market / rk_save_matrix_market,
rk_mm.cu) against the reference's own proj/src/matrix_market.cpp: written bytes
identical, loads identical, and every ParseError (message and line number)
identical on malformed files (proj/tests/sparse_core_test.cpp's cases and more)."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200.ranky import ParseError, load_matrix_market, save_matrix_market

pytestmark = pytest.mark.gpu

BANNER = "%%MatrixMarket matrix coordinate real general\n"


def ref_or_skip(ref):
    if ref.kind != "reference":
        pytest.skip("needs the reference build (oracle/_ref)")


def test_round_trip_bytes(ref, tmp_path):
    ref_or_skip(ref)
    for seed, (m, n, d) in enumerate([(64, 8192, 0.01), (7, 5, 0.5), (300, 2000, 0.02)]):
        a = configs.uniform(m, n, d, configs.VAL_NORMAL, seed)
        ours, theirs = tmp_path / f"o{seed}.mtx", tmp_path / f"r{seed}.mtx"
        save_matrix_market(a, ours)
        r, c, v = a.coo()
        ref.save_matrix_market((m, n, r, c, v), theirs)
        assert ours.read_bytes() == theirs.read_bytes()
        b = load_matrix_market(theirs)
        assert b == a
        rows, cols, rr, cc, vv = ref.load_matrix_market(ours)
        assert np.array_equal(rr, b.coo()[0]) and np.array_equal(cc, b.coo()[1]) and np.array_equal(vv, b.coo()[2])


def test_unsorted_and_blank_lines(ref, tmp_path):
    ref_or_skip(ref)
    p = tmp_path / "u.mtx"
    p.write_text(BANNER + "% comment\n3 4 4\n3 1 2.5\n\n1 4 -1e-300\r\n1 2 0.1\n2 2 7\n\n\n")
    a = load_matrix_market(p)
    rows, cols, r, c, v = ref.load_matrix_market(p)
    assert (a.rows(), a.cols()) == (rows, cols)
    assert np.array_equal(a.coo()[0], r) and np.array_equal(a.coo()[1], c) and np.array_equal(a.coo()[2], v)


BAD = {
    "empty": "",
    "header": "%%MatrixMarket matrix array real general\n1 1 1\n1 1 1\n",
    "no_dims": BANNER + "% only comments\n",
    "dims_extra": BANNER + "2 2 1 9\n1 1 1\n",
    "dims_bad": BANNER + "2 x 1\n1 1 1\n",
    "malformed": BANNER + "2 2 2\n1 1 1\n2 2\n",
    "value_bad": BANNER + "2 2 2\n1 1 1\n2 2 1.5q\n",
    "outside": BANNER + "2 2 2\n1 1 1\n3 1 1\n",
    "zero_index": BANNER + "2 2 2\n0 1 1\n1 1 1\n",
    "negative": BANNER + "2 2 1\n-1 1 1\n",
    "missing": BANNER + "3 3 3\n1 1 1\n2 2 2\n",
    "trailing": BANNER + "2 2 1\n1 1 1\n\n2 2 2\n",
    "duplicate": BANNER + "3 3 3\n2 2 1\n1 1 1\n2 2 5\n",
    "zero": BANNER + "2 2 2\n1 1 1\n2 2 0.0\n",
    "dup_and_zero": BANNER + "3 3 3\n1 1 0\n2 2 1\n2 2 5\n",
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_parse_errors_match_reference(case, ref, tmp_path):
    ref_or_skip(ref)
    from oracle import OracleError
    p = tmp_path / f"{case}.mtx"
    p.write_text(BAD[case])
    with pytest.raises(OracleError) as want:
        ref.load_matrix_market(p)
    with pytest.raises(ParseError) as got:
        load_matrix_market(p)
    assert want.value.code == 6  # the reference's ParseError
    assert str(got.value) == str(want.value)
    assert got.value.line == int(want.value.residual)


def test_many_chunks(ref, tmp_path):
    """enough lines for every parser thread to get a chunk; an error deep in the file"""
    ref_or_skip(ref)
    a = configs.uniform(500, 40000, 0.01, configs.VAL_NORMAL, 3)
    p = tmp_path / "big.mtx"
    save_matrix_market(a, p)
    assert load_matrix_market(p) == a
    lines = p.read_text().splitlines(keepends=True)
    lines[len(lines) * 3 // 4] = "12 13 abc\n"
    q = tmp_path / "big_bad.mtx"
    q.write_text("".join(lines))
    from oracle import OracleError
    with pytest.raises(OracleError) as want:
        ref.load_matrix_market(q)
    with pytest.raises(ParseError) as got:
        load_matrix_market(q)
    assert str(got.value) == str(want.value) and got.value.line == int(want.value.residual)
