"""Device ingestion of entries in any order (the reference's SparseMatrix
constructor sorts, then validates: proj/src/sparse_matrix.cpp:9-34): unsorted
input is radix-sorted on the device, so the pipeline result is bitwise the
sorted input's, and the first invalid entry in sorted order is reported with the
reference's message."""
import ctypes as C

import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200 import ranky as R

pytestmark = pytest.mark.gpu


def run_view(rows, cols, entries, cfg):
    e = np.ascontiguousarray(entries)
    v = R._View(rows, cols, len(e), e.ctypes.data_as(C.c_void_p))
    h = C.c_void_p()
    ctx = R.default_context()
    R._check(R.lib().rk_dev_matrix_create(ctx.handle, C.byref(v), C.byref(h)))
    dm = R.DeviceMatrix.__new__(R.DeviceMatrix)
    dm.ctx, dm._a, dm.handle, dm.rows, dm.cols, dm.nnz = ctx, None, h, rows, cols, len(e)
    out, _ = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
    try:
        sig, u, vv = R.dev_outputs_tensors(out)
        return sig.cpu().numpy(), u.cpu().numpy(), vv.cpu().numpy()
    finally:
        R.dev_outputs_free(out)
        dm.close()


def test_unsorted_entries_give_the_sorted_result():
    cfg = configs.CONFIGS["c2"]
    a = cfg.generate(4096 * 8)
    e = a.entries()
    cfg8 = configs.Config("c2", cfg.rows, a.cols(), 8, cfg.method, cfg.seed, 0, 0, "c2 slice")
    want = run_view(a.rows(), a.cols(), e, cfg8)
    shuffled = e[np.random.default_rng(3).permutation(len(e))]
    got = run_view(a.rows(), a.cols(), shuffled, cfg8)
    for x, y in zip(got, want):
        assert np.array_equal(x, y)


def test_unsorted_errors_report_the_first_in_sorted_order():
    e = np.zeros(4, dtype=R.ENTRY_DTYPE)
    e["row"] = [3, 0, 1, 0]
    e["col"] = [2, 5, 1, 5]
    e["value"] = [1.0, 2.0, 3.0, 4.0]
    with pytest.raises(R.InvalidArgument, match=r"duplicate sparse entry \(0, 5\)"):
        run_view(4, 8, e, configs.Config("x", 4, 8, 2, "none", 0, 0, 0, ""))
    e["col"] = [2, 5, 9, 6]  # (1, 9) outside 4x8 sorts before (3, 2)
    with pytest.raises(R.InvalidArgument, match=r"sparse entry \(1, 9\) outside 4x8"):
        run_view(4, 8, e, configs.Config("x", 4, 8, 2, "none", 0, 0, 0, ""))
