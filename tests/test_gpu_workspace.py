"""RepairWorkspace's single-row API on the device workspace (rk_workspace_*),
ported from the reference's proj/tests/repair_test.cpp: the brute-force
neighbor-set oracle (:16-40) over 40 instances (:127-146), the isolated-row and
no-in-block-candidate cases (:104-125), NeighborRandom (:148-175), and a replay
of the whole repair driver (proj/src/repair.cpp:162-216) through the single-row
API that must reproduce the batch repair -- and the reference's -- bit for bit."""
import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200.ranky import KeyedRng, RepairWorkspace

pytestmark = pytest.mark.gpu


def brute_force_neighbor_cols(a, p, d, row):
    """repair_test.cpp:16-40, straight from the definition."""
    dense = a.to_dense()
    rg = p.range(d)
    cand = set()
    for n1 in range(a.cols()):
        if rg.begin <= n1 < rg.end or dense[row, n1] == 0.0:
            continue
        cand |= {m for m in range(a.rows()) if dense[m, n1] != 0.0}
    return {n2 for m in cand for n2 in range(rg.begin, rg.end) if dense[m, n2] != 0.0}


def test_isolated_row_has_no_candidate():
    a = rk.SparseMatrix(3, 6, [(0, 0, 1.0), (2, 4, 1.0)])
    p = rk.partition_columns(6, 2)
    ws = RepairWorkspace(a, p)
    assert ws.apply_neighbor(0, 1, KeyedRng(3, 0, 1)) is None
    assert ws.to_matrix() == a


def test_candidates_without_in_block_columns():
    a = rk.SparseMatrix(4, 8, [(0, 5, 1.0), (1, 5, 1.0), (1, 6, 1.0), (2, 0, 1.0), (3, 2, 1.0)])
    p = rk.partition_columns(8, 2)
    assert rk.find_lonely_rows(a, p, 0) == [0, 1]
    assert brute_force_neighbor_cols(a, p, 0, 0) == set()
    ws = RepairWorkspace(a, p)
    assert ws.lonely_rows(0) == [0, 1]
    assert ws.apply_neighbor(0, 0, KeyedRng(3, 0, 0)) is None
    assert ws.to_matrix() == a


def test_neighbor_follows_shared_columns():
    # repair_test.cpp:90-102
    a = rk.SparseMatrix(3, 6, [(0, 0, 1.0), (0, 2, 1.0), (0, 5, 1.0), (1, 5, 1.0), (2, 1, 1.0)])
    p = rk.partition_columns(6, 2)
    ws = RepairWorkspace(a, p)
    col = ws.apply_neighbor(0, 1, KeyedRng(3, 0, 1))
    assert col in (0, 2)
    assert ws.has_entry(1, col) and not ws.row_lonely_in_block(0, 1)


def test_choice_matches_brute_force():
    # repair_test.cpp:127-146
    for instance in range(40):
        a = configs.synth_bipartite(8, 16, 0.12, instance)
        p = rk.partition_columns(16, 4)
        for d in range(4):
            for row in rk.find_lonely_rows(a, p, d):
                ws = RepairWorkspace(a, p)
                expected = brute_force_neighbor_cols(a, p, d, row)
                assert set(ws.neighbor_columns(d, row).tolist()) == expected
                col = ws.apply_neighbor(d, row, KeyedRng(instance, d, row))
                if not expected:
                    assert col is None
                else:
                    assert col in expected and ws.has_entry(row, col)


def test_neighbor_random_fills_the_row():
    a = rk.SparseMatrix(3, 6, [(0, 0, 1.0), (2, 4, 1.0)])
    p = rk.partition_columns(6, 2)
    ws = RepairWorkspace(a, p)
    assert len(ws.apply_neighbor_random(0, 1, KeyedRng(3, 0, 1))) == 1
    assert not ws.row_lonely_in_block(0, 1)
    a = rk.SparseMatrix(3, 6, [(0, 0, 1.0), (0, 2, 1.0), (0, 5, 1.0), (1, 5, 1.0), (2, 1, 1.0)])
    ws = RepairWorkspace(a, p)
    added = ws.apply_neighbor_random(0, 1, KeyedRng(3, 0, 1))
    assert 1 <= len(added) <= 2 and all(c < 3 and ws.has_entry(1, c) for c in added)
    assert not ws.row_lonely_in_block(0, 1)


def replay(a, p, method, seed):
    """proj/src/repair.cpp:162-216 driven through the single-row API."""
    ws = RepairWorkspace(a, p)
    edges, lonely, fallback = [], [], 0
    for d in range(p.block_count()):
        rows = ws.lonely_rows(d)
        lonely.append(len(rows))
        for row in rows:
            rng = KeyedRng(seed, d, row)
            if method == "random":
                edges.append((d, row, ws.apply_random(d, row, rng), 0))
            elif method == "neighbor":
                c = ws.apply_neighbor(d, row, rng)
                if c is None:
                    fallback += 1
                    edges.append((d, row, ws.apply_random(d, row, rng), 0))
                else:
                    edges.append((d, row, c, 1))
            else:
                c = ws.apply_neighbor(d, row, rng)
                if c is not None:
                    edges.append((d, row, c, 1))
                r = ws.apply_random(d, row, rng)
                if c is None or r != c:
                    edges.append((d, row, r, 0))
    return ws.to_matrix(), np.array(edges, dtype=np.int64).reshape(-1, 4), lonely, fallback


@pytest.mark.parametrize("method", ["random", "neighbor", "neighbor-random"])
def test_replay_equals_batch_repair_and_reference(method, ref):
    for seed in range(3):
        a = configs.synth_bipartite(16, 128, 0.05, seed)
        p = rk.partition_columns(128, 8)
        m, edges, lonely, fallback = replay(a, p, method, 17 + seed)
        rep, report = rk.repair(a, p, method, 17 + seed)
        assert m == rep
        assert np.array_equal(edges, report.edges_array())
        assert lonely == list(report.lonely_counts) and fallback == report.fallback_count
        r, c, v = a.coo()
        o = ref.repair((a.rows(), a.cols(), r, c, v), 8, method, 17 + seed)
        assert np.array_equal(edges, o.edges)
