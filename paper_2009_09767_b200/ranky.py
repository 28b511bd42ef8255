"""Python mirror of the reference's hot-path API (proj/include/ranky/*.hpp) on top
of the C ABI in include/ranky_b200.h (libranky_b200.so, sm_100a).

Names, argument meaning and error behaviour follow the reference:

=============================  ==================================================
reference (C++)                here
=============================  ==================================================
SparseMatrix / Entry           SparseMatrix (entries: ENTRY_DTYPE, same 24-byte layout)
partition_columns / block_view partition_columns / block_view
find_lonely_rows               find_lonely_rows        (GPU rank check)
repair / RepairReport          repair / RepairReport   (GPU checkers, bit-exact)
dense_svd / block_svd          dense_svd / block_svd   (GPU QR + Jacobi)
build_proxy / proxy_svd        build_proxy / proxy_svd
recover_right_vectors          recover_right_vectors   (GPU SpMM)
run_block_task                 run_block_task / run_block_tasks
proxy_from_records             proxy_from_records
run_pipeline / PipelineResult  run_pipeline / PipelineResult
std::invalid_argument          InvalidArgument (ValueError)
std::out_of_range              OutOfRange (IndexError)
ConvergenceError(residual)     ConvergenceError(.residual)
std::runtime_error             RankyRuntimeError (RuntimeError)
=============================  ==================================================

Every numeric routine runs on the GPU through the shared library; if the library
or a CUDA device is missing the call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libranky_b200.so")

ENTRY_DTYPE = np.dtype([("row", "<u8"), ("col", "<u8"), ("value", "<f8")])
K_RANK_TOL = 1e-10  # proj/include/ranky/svd.hpp:13


# ---------------------------------------------------------------------------
# errors (proj/include/ranky/errors.hpp:10-38 + the std:: types the reference throws)

class RankyError(Exception):
    pass


class InvalidArgument(RankyError, ValueError):
    pass


class OutOfRange(RankyError, IndexError):
    pass


class ConvergenceError(RankyError, RuntimeError):
    def __init__(self, what: str, residual: float):
        super().__init__(what)
        self.residual = residual


class RankyRuntimeError(RankyError, RuntimeError):
    pass


GRAM_REJECTED = 8  # rk_status RK_GRAM_REJECTED


class GramRejected(RankyError):
    """RK_GRAM_REJECTED: the sharded merge's Gram route does not apply; the caller
    takes the TSQR path (rk_dev_shard_tsqr, all-gather, rk_dev_shard_finish)."""


class ParseError(RankyError, RuntimeError):
    """ranky::ParseError (proj/include/ranky/errors.hpp:9-20): message "... (line L)", .line"""

    def __init__(self, message: str, line: int = 0):
        super().__init__(message)
        self.line = line


class RecordError(RankyError, RuntimeError):
    """ranky::RecordError (proj/include/ranky/errors.hpp:23-26): damaged block record"""


class CudaError(RankyError, RuntimeError):
    pass


class RepairMethod(IntEnum):
    """proj/include/ranky/repair.hpp:15-20"""
    kRandom = 0
    kNeighbor = 1
    kNeighborRandom = 2
    kNone = 3


_METHOD_NAMES = {RepairMethod.kRandom: "random", RepairMethod.kNeighbor: "neighbor",
                 RepairMethod.kNeighborRandom: "neighbor-random", RepairMethod.kNone: "none"}


def to_string(method: RepairMethod) -> str:
    """repair.cpp:9-17"""
    return _METHOD_NAMES[RepairMethod(method)]


def repair_method_from_string(name: str) -> RepairMethod:
    """repair.cpp:19-25"""
    for m, n in _METHOD_NAMES.items():
        if n == name:
            return m
    raise InvalidArgument(f"unknown repair method '{name}'")


def _method(m) -> int:
    if isinstance(m, str):
        return int(repair_method_from_string(m))
    return int(RepairMethod(m))


# ---------------------------------------------------------------------------
# ctypes binding

class _View(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64), ("entries", C.c_void_p)]


class _Svd(C.Structure):
    _fields_ = [("u_rows", C.c_uint64), ("u_cols", C.c_uint64), ("u", C.POINTER(C.c_double)),
                ("n_sigma", C.c_uint64), ("sigma", C.POINTER(C.c_double)), ("has_v", C.c_int32),
                ("v_rows", C.c_uint64), ("v_cols", C.c_uint64), ("v", C.POINTER(C.c_double))]


class _Report(C.Structure):
    _fields_ = [("n_edges", C.c_uint64), ("block", C.POINTER(C.c_uint64)), ("row", C.POINTER(C.c_uint64)),
                ("col", C.POINTER(C.c_uint64)), ("mechanism", C.POINTER(C.c_int32)),
                ("n_blocks", C.c_uint64), ("lonely_counts", C.POINTER(C.c_uint64)), ("fallback_count", C.c_uint64)]


class _Sparse(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64), ("entries", C.c_void_p)]


class _Records(C.Structure):
    _fields_ = [("n_records", C.c_uint64), ("rows", C.c_uint64), ("kept", C.POINTER(C.c_uint32)),
                ("offset", C.POINTER(C.c_uint64)), ("payload", C.POINTER(C.c_double))]


class Timing(C.Structure):
    _fields_ = [("repair_ms", C.c_double), ("blocks_ms", C.c_double), ("merge_ms", C.c_double),
                ("recover_ms", C.c_double), ("total_ms", C.c_double), ("qr_ms", C.c_double),
                ("jacobi_ms", C.c_double), ("jacobi_sweeps_max", C.c_uint64), ("jacobi_rotations", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("jacobi_sweeps_sum", C.c_uint64), ("qr_flops", C.c_double),
                ("jacobi_flops", C.c_double), ("merge_sweeps", C.c_uint64), ("merge_rotations", C.c_uint64),
                ("merge_flops", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class _Pipeline(C.Structure):
    _fields_ = [("svd", _Svd), ("report", _Report), ("repaired", _Sparse), ("records", _Records),
                ("timing", Timing)]


class DevOutputs(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("k_sigma", C.c_uint64), ("k_v", C.c_uint64),
                ("d_sigma", C.c_void_p), ("d_u", C.c_void_p), ("d_v", C.c_void_p), ("n_edges", C.c_uint64)]


WANT_V, WANT_REPAIRED, WANT_RECORDS = 1, 2, 4

_lib = None
# rk_allgather_fn: (user, const double* d_mine, double* d_all, uint64_t count)
ALLGATHER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
_lib_lock = threading.Lock()


def lib():
    """Load libranky_b200.so (raises if it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with paper_2009_09767_b200._build.build()")
        L = C.CDLL(LIB_PATH)
        u64, i32, u32, dbl, vp = C.c_uint64, C.c_int32, C.c_uint32, C.c_double, C.c_void_p
        pu64, pdbl = C.POINTER(C.c_uint64), C.POINTER(C.c_double)
        sig = {
            "rk_last_error": ([], C.c_char_p), "rk_last_residual": ([], dbl), "rk_abi_version": ([], i32),
            "rk_reload_tuning": ([], None), "rk_build_flags": ([], u32), "rk_last_error_line": ([], u64),
            "rk_load_matrix_market": ([vp, C.c_char_p, C.POINTER(_Sparse)], i32),
            "rk_save_matrix_market": ([C.POINTER(_View), C.c_char_p], i32),
            "rk_multi_create": ([C.POINTER(C.c_int32), u32, C.POINTER(vp)], i32),
            "rk_multi_destroy": ([vp], i32),
            "rk_multi_run_pipeline": ([vp, C.POINTER(_View), u64, i32, u64, u64, u32, u64, C.POINTER(_Pipeline)],
                                      i32),
            "rk_nccl_unique_id": ([C.POINTER(C.c_uint8)], i32),
            "rk_dist_create": ([vp, i32, i32, C.POINTER(C.c_uint8), C.POINTER(vp)], i32),
            "rk_dist_destroy": ([vp], i32),
            "rk_dist_full_svd": ([vp, vp, u64, i32, u64, u64, u32, u64, C.POINTER(C.POINTER(DevOutputs)),
                                  C.POINTER(Timing), pu64, pu64], i32),
            "rk_dev_sharded_full_svd": ([vp, vp, u64, i32, u64, u64, u32, u64, i32, i32, ALLGATHER_FN, vp,
                                         C.POINTER(C.POINTER(DevOutputs)), C.POINTER(Timing), pu64, pu64], i32),
            "rk_workspace_create": ([vp, C.POINTER(_View), u64, C.POINTER(vp)], i32),
            "rk_workspace_destroy": ([vp], i32),
            "rk_workspace_has_entry": ([vp, u64, u64, C.POINTER(C.c_int32)], i32),
            "rk_workspace_row_lonely_in_block": ([vp, u64, u64, C.POINTER(C.c_int32)], i32),
            "rk_workspace_lonely_rows": ([vp, u64, pu64, pu64], i32),
            "rk_workspace_neighbor_columns": ([vp, u64, u64, pu64, pu64], i32),
            "rk_workspace_insert": ([vp, u64, u64], i32),
            "rk_workspace_to_matrix": ([vp, C.POINTER(_Sparse)], i32),
            "rk_sigma_error": ([vp, pdbl, u64, pdbl, u64, pdbl], i32),
            "rk_align_signs": ([vp, pdbl, pdbl, u64, u64, pdbl, u64, pdbl], i32),
            "rk_left_vector_error": ([vp, pdbl, pdbl, u64, u64, pdbl, u64, pdbl], i32),
            "rk_numerical_rank": ([vp, pdbl, u64, u64, dbl, pu64], i32),
            "rk_dev_sigma_error": ([vp, vp, u64, vp, u64, pdbl], i32),
            "rk_dev_align_signs": ([vp, vp, vp, u64, u64, vp, u64, vp], i32),
            "rk_dev_left_vector_error": ([vp, vp, vp, u64, u64, vp, u64, pdbl], i32),
            "rk_dev_numerical_rank": ([vp, vp, u64, u64, dbl, pu64], i32),
            "rk_ctx_create": ([i32, C.POINTER(vp)], i32), "rk_ctx_destroy": ([vp], i32),
            "rk_ctx_set_stream": ([vp, vp], i32), "rk_ctx_synchronize": ([vp], i32),
            "rk_ctx_kernel_launches": ([vp], u64),
            "rk_svd_free": ([C.POINTER(_Svd)], None), "rk_host_free": ([C.c_void_p], None), "rk_repair_report_free": ([C.POINTER(_Report)], None),
            "rk_sparse_free": ([C.POINTER(_Sparse)], None), "rk_records_free": ([C.POINTER(_Records)], None),
            "rk_pipeline_result_free": ([C.POINTER(_Pipeline)], None),
            "rk_keyed_rng_next": ([vp, u64, u64, pu64, pu64, u64, pu64], i32),
            "rk_keyed_rng_below": ([vp, u64, u64, pu64, pu64, pu64, pu64], i32),
            "rk_find_lonely_rows": ([vp, C.POINTER(_View), u64, u64, pu64, pu64], i32),
            "rk_repair": ([vp, C.POINTER(_View), u64, i32, u64, C.POINTER(_Sparse), C.POINTER(_Report)], i32),
            "rk_dense_svd": ([vp, u64, u64, pdbl, C.POINTER(_Svd)], i32),
            "rk_block_svd": ([vp, C.POINTER(_View), u64, C.POINTER(_Svd)], i32),
            "rk_proxy_svd": ([vp, u64, u64, pdbl, u64, pu64, C.POINTER(_Svd)], i32),
            "rk_recover_right_vectors": ([vp, C.POINTER(_View), u64, u64, pdbl, u64, pdbl, dbl,
                                          C.POINTER(_Svd)], i32),
            "rk_run_block_tasks": ([vp, C.POINTER(_View), u64, u64, C.POINTER(_Records)], i32),
            "rk_run_pipeline": ([vp, C.POINTER(_View), u64, i32, u64, u64, u64, u32, u64,
                                 C.POINTER(_Pipeline)], i32),
            "rk_dev_matrix_create": ([vp, C.POINTER(_View), C.POINTER(vp)], i32),
            "rk_dev_matrix_destroy": ([vp], i32), "rk_dev_matrix_nnz": ([vp], u64),
            "rk_dev_full_svd": ([vp, vp, u64, i32, u64, u64, u32, u64, C.POINTER(C.POINTER(DevOutputs)),
                                 C.POINTER(Timing)], i32),
            "rk_dev_outputs_free": ([C.POINTER(DevOutputs)], i32),
            "rk_dev_residual": ([vp, vp, C.POINTER(DevOutputs), pdbl, pdbl], i32),
            "rk_crc32": ([vp, u64], u32),
            "rk_dev_crc32": ([vp, vp, pu64, pu64, u64, C.POINTER(C.c_uint32)], i32),
            "rk_write_block_record": ([u32, u32, u32, pdbl, C.c_char_p], i32),
            "rk_read_block_record": ([C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(pdbl)], i32),
            "rk_write_records": ([vp, C.POINTER(_Records), C.c_char_p], i32),
            "rk_merge_tree_leaves": ([u64, u64, u64, u64], u64),
            "rk_dev_shard_factor": ([vp, vp, u64, i32, u64, u64, u64, u64, vp, C.POINTER(vp), C.POINTER(Timing)],
                                    i32),
            "rk_dev_shard_finish": ([vp, vp, vp, u64, u32, u64, u64, u64, C.POINTER(C.POINTER(DevOutputs)),
                                     C.POINTER(Timing)], i32),
            "rk_dev_shard_destroy": ([vp], i32),
            "rk_dev_shard_factor_gram": ([vp, vp, u64, i32, u64, u64, u64, u64, vp, C.POINTER(vp),
                                          C.POINTER(Timing)], i32),
            "rk_dev_shard_finish_gram": ([vp, vp, vp, u64, u32, u64, u64, u64, C.POINTER(C.POINTER(DevOutputs)),
                                          C.POINTER(Timing)], i32),
            "rk_dev_shard_tsqr": ([vp, vp, vp], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
        return L


def reload_tuning() -> None:
    """Re-read the RK_* tuning switches (the library reads them once per process)."""
    lib().rk_reload_tuning()


def experiments_built() -> bool:
    """True when libranky_b200.so is the experiments build (RK_EXPERIMENTS=1)."""
    return bool(lib().rk_build_flags() & 1)


def _check(status: int):
    if status == 0:
        return
    L = lib()
    msg = L.rk_last_error().decode(errors="replace")
    if status == 1:
        raise InvalidArgument(msg)
    if status == 2:
        raise OutOfRange(msg)
    if status == 3:
        raise ConvergenceError(msg, L.rk_last_residual())
    if status == 4:
        raise RankyRuntimeError(msg)
    if status == 5:
        raise CudaError(msg)
    if status == 6:
        raise MemoryError(msg)
    if status == 7:
        raise RecordError(msg)
    if status == GRAM_REJECTED:
        raise GramRejected(msg)
    if status == 9:
        raise ParseError(msg, int(L.rk_last_error_line()))
    raise RankyError(f"status {status}: {msg}")


class Context:
    """One CUDA device + stream (rk_ctx)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.rk_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib().rk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        _check(lib().rk_ctx_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        _check(lib().rk_ctx_synchronize(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(lib().rk_ctx_kernel_launches(self.handle))


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("RANKY_DEVICE", "0")))
        _tls.ctx = ctx
    return ctx


def _ctx(ctx):
    return (ctx or default_context()).handle


# ---------------------------------------------------------------------------
# containers

class SparseMatrix:
    """Immutable COO matrix sorted by (row, col) -- proj/src/sparse_matrix.cpp:9-34.

    Construction validates like the reference: out-of-range index, stored zero
    and duplicate entries raise InvalidArgument.
    """

    def __init__(self, rows: int, cols: int, entries=None):
        self._rows, self._cols = int(rows), int(cols)
        if entries is None:
            e = np.zeros(0, dtype=ENTRY_DTYPE)
        elif isinstance(entries, np.ndarray) and entries.dtype == ENTRY_DTYPE:
            e = entries.copy()
        elif isinstance(entries, tuple) and len(entries) == 3:
            r, c, v = entries
            e = np.zeros(len(r), dtype=ENTRY_DTYPE)
            e["row"], e["col"], e["value"] = r, c, v
        else:
            lst = list(entries)
            e = np.zeros(len(lst), dtype=ENTRY_DTYPE)
            for i, (r, c, v) in enumerate(lst):
                e[i] = (r, c, v)
        order = np.lexsort((e["col"], e["row"]))
        e = e[order]
        if len(e):
            # the reference checks entry by entry in sorted order (sparse_matrix.cpp:15-29):
            # the first entry that violates any rule decides which error is raised
            out = (e["row"] >= self._rows) | (e["col"] >= self._cols)
            zero = e["value"] == 0.0
            dup = np.zeros(len(e), dtype=bool)
            dup[1:] = (e["row"][1:] == e["row"][:-1]) & (e["col"][1:] == e["col"][:-1])
            bad = out | zero | dup
            if bad.any():
                i = int(np.argmax(bad))
                if out[i]:
                    raise InvalidArgument(f"sparse entry ({e['row'][i]}, {e['col'][i]}) outside {rows}x{cols}")
                if zero[i]:
                    raise InvalidArgument(f"sparse entry ({e['row'][i]}, {e['col'][i]}) stores zero")
                raise InvalidArgument(f"duplicate sparse entry ({e['row'][i]}, {e['col'][i]})")
        self._e = np.ascontiguousarray(e)

    @classmethod
    def _trusted(cls, rows, cols, entries: np.ndarray) -> "SparseMatrix":
        m = cls.__new__(cls)
        m._rows, m._cols, m._e = int(rows), int(cols), np.ascontiguousarray(entries)
        return m

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nnz(self) -> int:
        return len(self._e)

    def entries(self) -> np.ndarray:
        return self._e

    def row_entries(self, row: int) -> np.ndarray:
        if row >= self._rows:
            raise OutOfRange(f"row {row}")
        lo = np.searchsorted(self._e["row"], row, "left")
        hi = np.searchsorted(self._e["row"], row, "right")
        return self._e[lo:hi]

    def count_in_columns(self, row: int, col_begin: int, col_end: int) -> int:
        re = self.row_entries(row)
        return int(np.count_nonzero((re["col"] >= col_begin) & (re["col"] < col_end)))

    def coo(self):
        return self._e["row"].copy(), self._e["col"].copy(), self._e["value"].copy()

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self._rows, self._cols))
        a[self._e["row"].astype(np.int64), self._e["col"].astype(np.int64)] = self._e["value"]
        return a

    def _view(self) -> _View:
        return _View(self._rows, self._cols, len(self._e), self._e.ctypes.data if len(self._e) else None)

    def __eq__(self, other):
        return (isinstance(other, SparseMatrix) and self._rows == other._rows and self._cols == other._cols
                and np.array_equal(self._e, other._e))

    def __repr__(self):
        return f"SparseMatrix({self._rows}x{self._cols}, nnz={len(self._e)})"


def sparse_of(a: np.ndarray) -> SparseMatrix:
    """proj/src/dense_matrix.cpp:77-83"""
    a = np.asarray(a, dtype=np.float64)
    r, c = np.nonzero(a)
    return SparseMatrix._trusted(a.shape[0], a.shape[1], _entries(r, c, a[r, c]))


def _entries(r, c, v) -> np.ndarray:
    e = np.zeros(len(r), dtype=ENTRY_DTYPE)
    e["row"], e["col"], e["value"] = r, c, v
    return e


@dataclass(frozen=True)
class ColumnRange:
    begin: int
    end: int

    def width(self) -> int:
        return self.end - self.begin


class BlockPartition:
    """proj/include/ranky/partition.hpp:22-41"""

    def __init__(self, total_cols: int, ranges: list[ColumnRange]):
        expect = 0
        for r in ranges:
            if r.begin != expect or r.end <= r.begin:
                raise InvalidArgument("partition ranges must be contiguous and nonempty")
            expect = r.end
        if expect != total_cols:
            raise InvalidArgument("partition ranges must cover all columns")
        self._total, self._ranges = total_cols, list(ranges)

    def total_cols(self) -> int:
        return self._total

    def block_count(self) -> int:
        return len(self._ranges)

    def range(self, d: int) -> ColumnRange:
        if d >= len(self._ranges):
            raise OutOfRange(f"block index {d} of {len(self._ranges)}")
        return self._ranges[d]

    def ranges(self):
        return list(self._ranges)

    def block_of(self, col: int) -> int:
        if col >= self._total:
            raise OutOfRange(f"column {col}")
        ends = [r.end for r in self._ranges]
        return int(np.searchsorted(ends, col, side="right"))

    def __eq__(self, other):
        return isinstance(other, BlockPartition) and self._total == other._total and self._ranges == other._ranges


def partition_columns(n_cols: int, block_count: int) -> BlockPartition:
    """proj/src/partition.cpp:38-51"""
    if block_count == 0 or block_count > n_cols:
        raise InvalidArgument(f"cannot split {n_cols} columns into {block_count} blocks")
    w = n_cols // block_count
    return BlockPartition(n_cols, [ColumnRange(d * w, n_cols if d + 1 == block_count else (d + 1) * w)
                                   for d in range(block_count)])


def _is_uniform(p: BlockPartition) -> bool:
    ref = partition_columns(p.total_cols(), p.block_count())
    return ref == p


def block_view(a: SparseMatrix, p: BlockPartition, d: int) -> SparseMatrix:
    """proj/src/partition.cpp:53-62 (host-side slicing of the container)"""
    rg = p.range(d)
    e = a.entries()
    m = (e["col"] >= rg.begin) & (e["col"] < rg.end)
    sub = e[m].copy()
    sub["col"] -= rg.begin
    return SparseMatrix._trusted(a.rows(), rg.width(), sub)


# ---------------------------------------------------------------------------
# repair

@dataclass
class AddedEdge:
    block: int
    row: int
    col: int
    mechanism: RepairMethod = RepairMethod.kRandom


@dataclass
class RepairReport:
    """proj/include/ranky/repair.hpp:38-48"""
    added_edges: list = field(default_factory=list)
    lonely_counts: list = field(default_factory=list)
    fallback_count: int = 0

    def to_log(self) -> str:
        """repair.cpp:27-40"""
        out = [f"{e.block}\t{e.row}\t{e.col}\t{to_string(e.mechanism)}\n" for e in self.added_edges]
        out.append("# lonely=" + ",".join(str(x) for x in self.lonely_counts) + f" fallback={self.fallback_count}\n")
        return "".join(out)

    def edges_array(self) -> np.ndarray:
        a = np.zeros((len(self.added_edges), 4), dtype=np.int64)
        for i, e in enumerate(self.added_edges):
            a[i] = (e.block, e.row, e.col, 1 if e.mechanism == RepairMethod.kNeighbor else 0)
        return a


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True)


def _report_of(r: _Report) -> RepairReport:
    n = int(r.n_edges)
    b, rw, c, m = (_arr(r.block, n, np.int64), _arr(r.row, n, np.int64), _arr(r.col, n, np.int64),
                   _arr(r.mechanism, n, np.int64))
    edges = [AddedEdge(int(b[i]), int(rw[i]), int(c[i]), RepairMethod.kNeighbor if m[i] else RepairMethod.kRandom)
             for i in range(n)]
    return RepairReport(edges, [int(x) for x in _arr(r.lonely_counts, r.n_blocks, np.int64)], int(r.fallback_count))


def _sparse_of(s: _Sparse) -> SparseMatrix:
    """The library's entry array as the matrix's storage (no copy)."""
    n = int(s.nnz)
    e = _take_array(s, "entries", n, (n,), ENTRY_DTYPE) if n else np.zeros(0, dtype=ENTRY_DTYPE)
    return SparseMatrix._trusted(s.rows, s.cols, e)


def _uniform_or_raise(a: SparseMatrix, p: BlockPartition):
    if p.total_cols() != a.cols():
        raise InvalidArgument("partition does not match matrix columns")
    if not _is_uniform(p):
        raise InvalidArgument("only partitions made by partition_columns are supported")


def find_lonely_rows(a: SparseMatrix, p: BlockPartition, d: int, ctx: Context | None = None) -> list[int]:
    """proj/src/repair.cpp:42-50 (GPU scan)"""
    _uniform_or_raise(a, p)
    out = np.zeros(max(a.rows(), 1), dtype=np.uint64)
    n = C.c_uint64()
    v = a._view()
    _check(lib().rk_find_lonely_rows(_ctx(ctx), C.byref(v), p.block_count(), d,
                                     out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(n)))
    return [int(x) for x in out[:n.value]]


def repair(a: SparseMatrix, p: BlockPartition, method, seed: int, ctx: Context | None = None):
    """proj/src/repair.cpp:162-216 -> (repaired SparseMatrix, RepairReport)"""
    _uniform_or_raise(a, p)
    v = a._view()
    sp, rep = _Sparse(), _Report()
    L = lib()
    st = L.rk_repair(_ctx(ctx), C.byref(v), p.block_count(), _method(method), seed, C.byref(sp), C.byref(rep))
    try:
        _check(st)
        return _sparse_of(sp), _report_of(rep)
    finally:
        L.rk_sparse_free(C.byref(sp))
        L.rk_repair_report_free(C.byref(rep))


def rank_equal_probability(columns: int, single_entry_rows: int) -> float:
    """Eq. (5) -- proj/src/repair.cpp:218-223 (host arithmetic, no kernel)"""
    if columns == 0:
        raise InvalidArgument("column count must be positive")
    if single_entry_rows >= columns:
        return 0.0
    return (columns - single_entry_rows) / columns


def keyed_rng_next(seed: int, block, row, draws: int, ctx: Context | None = None) -> np.ndarray:
    """KeyedRng::next streams evaluated on the device -- proj/src/rng.cpp:16-25"""
    b = np.ascontiguousarray(np.atleast_1d(block), dtype=np.uint64)
    r = np.ascontiguousarray(np.atleast_1d(row), dtype=np.uint64)
    out = np.zeros((len(b), draws), dtype=np.uint64)
    p = C.POINTER(C.c_uint64)
    _check(lib().rk_keyed_rng_next(_ctx(ctx), len(b), seed, b.ctypes.data_as(p), r.ctypes.data_as(p), draws,
                                   out.ctypes.data_as(p)))
    return out


def keyed_rng_below(seed: int, block, row, bound, ctx: Context | None = None) -> np.ndarray:
    """KeyedRng::below on the device -- proj/src/rng.cpp:27-34"""
    b = np.ascontiguousarray(np.atleast_1d(block), dtype=np.uint64)
    r = np.ascontiguousarray(np.atleast_1d(row), dtype=np.uint64)
    bd = np.ascontiguousarray(np.broadcast_to(np.atleast_1d(bound), b.shape), dtype=np.uint64)
    out = np.zeros(len(b), dtype=np.uint64)
    p = C.POINTER(C.c_uint64)
    _check(lib().rk_keyed_rng_below(_ctx(ctx), len(b), seed, b.ctypes.data_as(p), r.ctypes.data_as(p),
                                    bd.ctypes.data_as(p), out.ctypes.data_as(p)))
    return out


_M64 = (1 << 64) - 1


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class KeyedRng:
    """The reference's generator object (proj/include/ranky/rng.hpp:11-25,
    proj/src/rng.cpp:8-38): a caller-owned splitmix64 stream keyed by (seed, block,
    row). RepairWorkspace draws from it on the host, as the reference does; the
    batch repair evaluates the same streams on the device (keyed_rng_*)."""

    def __init__(self, seed: int, block: int, row: int):
        st = _mix((seed + 0x9E3779B97F4A7C15) & _M64)
        st = _mix(st ^ ((block + 0xBF58476D1CE4E5B9) & _M64))
        self.state = _mix(st ^ ((row + 0x94D049BB133111EB) & _M64))

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        return _mix(self.state)

    def below(self, bound: int) -> int:
        threshold = ((1 << 64) - bound) % bound
        while True:
            r = self.next()
            if r >= threshold:
                return r % bound

    def unit(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53


class RepairWorkspace:
    """RepairWorkspace (proj/include/ranky/repair.hpp:56-87, proj/src/repair.cpp:52-160)
    on a device workspace (rk_workspace_*: the matrix's CSR + CSC in HBM plus the
    inserted edges). The neighbor scan runs on the device; the draws come from the
    caller's KeyedRng on the host, where the reference makes them."""

    def __init__(self, a: SparseMatrix, p: BlockPartition, ctx: Context | None = None):
        if p.total_cols() != a.cols():
            raise InvalidArgument("partition does not match matrix columns")
        _uniform_or_raise(a, p)
        self._a, self._p, self._ctx = a, p, ctx
        self._h = C.c_void_p()
        v = a._view()
        _check(lib().rk_workspace_create(_ctx(ctx), C.byref(v), p.block_count(), C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.rk_workspace_destroy(h)
            self._h = C.c_void_p()

    def _insert(self, row: int, col: int) -> None:
        _check(lib().rk_workspace_insert(self._h, row, col))

    def apply_random(self, d: int, row: int, rng: KeyedRng) -> int:
        """repair.cpp:95-101"""
        rg = self._p.range(d)
        col = rg.begin + rng.below(rg.end - rg.begin)
        self._insert(row, col)
        return col

    def neighbor_columns(self, d: int, row: int) -> np.ndarray:
        """The NeighborChecker's candidate columns before the draw (repair.cpp:107-125)."""
        rg = self._p.range(d)
        out = np.zeros(max(1, rg.end - rg.begin), dtype=np.uint64)
        n = C.c_uint64()
        p = C.POINTER(C.c_uint64)
        _check(lib().rk_workspace_neighbor_columns(self._h, d, row, out.ctypes.data_as(p), C.byref(n)))
        return out[:n.value].astype(np.int64)

    def apply_neighbor(self, d: int, row: int, rng: KeyedRng):
        """repair.cpp:103-135: None (no draw, no edge) when no candidate column exists."""
        cols = self.neighbor_columns(d, row)
        if len(cols) == 0:
            return None
        col = int(cols[rng.below(len(cols))])
        self._insert(row, col)
        return col

    def apply_neighbor_random(self, d: int, row: int, rng: KeyedRng) -> list[int]:
        """repair.cpp:137-145"""
        added = []
        c = self.apply_neighbor(d, row, rng)
        if c is not None:
            added.append(c)
        rc = self.apply_random(d, row, rng)
        if not added or added[0] != rc:
            added.append(rc)
        return added

    def has_entry(self, row: int, col: int) -> bool:
        out = C.c_int32()
        _check(lib().rk_workspace_has_entry(self._h, row, col, C.byref(out)))
        return bool(out.value)

    def row_lonely_in_block(self, d: int, row: int) -> bool:
        out = C.c_int32()
        _check(lib().rk_workspace_row_lonely_in_block(self._h, d, row, C.byref(out)))
        return bool(out.value)

    def lonely_rows(self, d: int) -> list[int]:
        out = np.zeros(max(1, self._a.rows()), dtype=np.uint64)
        n = C.c_uint64()
        _check(lib().rk_workspace_lonely_rows(self._h, d, out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def to_matrix(self) -> SparseMatrix:
        out = _Sparse()
        st = lib().rk_workspace_to_matrix(self._h, C.byref(out))
        try:
            _check(st)
            return _sparse_of(out)
        finally:
            lib().rk_sparse_free(C.byref(out))


# ---------------------------------------------------------------------------
# SVD

@dataclass
class SvdResult:
    """proj/include/ranky/svd.hpp:15-19"""
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray | None = None


class _HostBuffer:
    """Owns one library-allocated host buffer; numpy arrays view it without a copy."""

    def __init__(self, addr):
        self.addr = addr

    def __del__(self):
        try:
            lib().rk_host_free(C.c_void_p(self.addr))
        except Exception:
            pass


def _take_array(struct, field: str, n: int, shape, dtype=np.float64) -> np.ndarray:
    """Zero-copy numpy view of a large result buffer; ownership moves to the array
    (the struct field is cleared so the record's free does not release it)."""
    ptr = getattr(struct, field)
    addr = ptr if (ptr is None or isinstance(ptr, int)) else C.cast(ptr, C.c_void_p).value
    dtype = np.dtype(dtype)
    if n < (1 << 17) or not addr:
        if not addr or n == 0:
            return np.zeros(shape, dtype=dtype)
        raw = (C.c_char * (n * dtype.itemsize)).from_address(addr)
        return np.frombuffer(raw, dtype=dtype).copy().reshape(shape)
    buf = (C.c_char * (n * dtype.itemsize)).from_address(addr)
    arr = np.frombuffer(buf, dtype=dtype).reshape(shape)
    keeper = _HostBuffer(addr)
    setattr(struct, field, None if isinstance(ptr, int) else C.cast(C.c_void_p(0), type(ptr)))
    holder = np.ndarray.__new__(_Owned, arr.shape, dtype=arr.dtype, buffer=buf)
    holder._keeper = keeper
    return holder


class _Owned(np.ndarray):
    """ndarray subclass that keeps the library buffer alive."""


def _svd_of(s: _Svd) -> SvdResult:
    u = _take_array(s, "u", int(s.u_rows * s.u_cols), (int(s.u_rows), int(s.u_cols)))
    sig = _arr(s.sigma, s.n_sigma, np.float64)
    v = None
    if s.has_v:
        v = _take_array(s, "v", int(s.v_rows * s.v_cols), (int(s.v_rows), int(s.v_cols)))
    return SvdResult(u, sig, v)


def dense_svd(a: np.ndarray, ctx: Context | None = None) -> SvdResult:
    """proj/src/svd.cpp:365-379 (GPU: QR + one-sided Jacobi + apply_q)"""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise InvalidArgument("dense_svd: expected a matrix")
    out = _Svd()
    L = lib()
    st = L.rk_dense_svd(_ctx(ctx), a.shape[0], a.shape[1], a.ctypes.data_as(C.POINTER(C.c_double)), C.byref(out))
    try:
        _check(st)
        return _svd_of(out)
    finally:
        L.rk_svd_free(C.byref(out))


def block_svd(block: SparseMatrix, keep: int, ctx: Context | None = None) -> SvdResult:
    """proj/src/svd.cpp:381-400 (GPU: compaction + QR + Jacobi); v is None"""
    v = block._view()
    out = _Svd()
    L = lib()
    st = L.rk_block_svd(_ctx(ctx), C.byref(v), keep, C.byref(out))
    try:
        _check(st)
        r = _svd_of(out)
        return SvdResult(r.u, r.sigma, None)
    finally:
        L.rk_svd_free(C.byref(out))


@dataclass
class ProxyMatrix:
    """proj/include/ranky/proxy.hpp:13-16"""
    matrix: np.ndarray
    block_offsets: list


def build_proxy(block_results, rows: int) -> ProxyMatrix:
    """proj/src/proxy.cpp:8-38 -- concatenation of U*Sigma (host container assembly)"""
    total = 0
    for r in block_results:
        if r.u.shape[0] != rows:
            raise InvalidArgument(f"build_proxy: block factor has {r.u.shape[0]} rows, expected {rows}")
        if r.u.shape[1] != len(r.sigma):
            raise InvalidArgument("build_proxy: U column count does not match sigma")
        total += len(r.sigma)
    m = np.zeros((rows, total))
    offs, off = [], 0
    for r in block_results:
        offs.append(off)
        k = len(r.sigma)
        m[:, off:off + k] = r.u * np.asarray(r.sigma)[None, :]
        off += k
    offs.append(off)
    return ProxyMatrix(m, offs)


def proxy_svd(proxy: ProxyMatrix, ctx: Context | None = None) -> SvdResult:
    """proj/src/proxy.cpp:40-46"""
    m = np.ascontiguousarray(proxy.matrix, dtype=np.float64)
    offs = np.ascontiguousarray(proxy.block_offsets, dtype=np.uint64)
    out = _Svd()
    L = lib()
    st = L.rk_proxy_svd(_ctx(ctx), m.shape[0], m.shape[1], m.ctypes.data_as(C.POINTER(C.c_double)), len(offs),
                        offs.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(out))
    try:
        _check(st)
        return _svd_of(out)
    finally:
        L.rk_svd_free(C.byref(out))


def recover_right_vectors(a: SparseMatrix, u: np.ndarray, sigma, tol: float = K_RANK_TOL,
                          ctx: Context | None = None) -> np.ndarray:
    """proj/src/proxy.cpp:48-72 (GPU SpMM, bit-exact given U and sigma)"""
    u = np.ascontiguousarray(u, dtype=np.float64)
    s = np.ascontiguousarray(sigma, dtype=np.float64)
    v = a._view()
    out = _Svd()
    L = lib()
    st = L.rk_recover_right_vectors(_ctx(ctx), C.byref(v), u.shape[0], u.shape[1],
                                    u.ctypes.data_as(C.POINTER(C.c_double)), len(s),
                                    s.ctypes.data_as(C.POINTER(C.c_double)), tol, C.byref(out))
    try:
        _check(st)
        return _svd_of(out).v
    finally:
        L.rk_svd_free(C.byref(out))


# ---------------------------------------------------------------------------
# Matrix Market -- proj/src/matrix_market.cpp:38-132 (rk_mm.cu)

def load_matrix_market(path, ctx: Context | None = None) -> SparseMatrix:
    """The reference's loader: same header/dimension/entry rules and ParseError
    messages with line numbers; entries sorted on the device."""
    out = _Sparse()
    L = lib()
    st = L.rk_load_matrix_market(_ctx(ctx), str(path).encode(), C.byref(out))
    try:
        _check(st)
        return _sparse_of(out)
    finally:
        L.rk_sparse_free(C.byref(out))


def save_matrix_market(a: SparseMatrix, path) -> None:
    """Byte-identical to the reference's writer (shortest round-trip values)."""
    v = a._view()
    _check(lib().rk_save_matrix_market(C.byref(v), str(path).encode()))


# ---------------------------------------------------------------------------
# evaluation metrics -- proj/include/ranky/metrics.hpp, proj/src/metrics.cpp:32-114 (rk_eval.cu)

def _pd(x):
    return x.ctypes.data_as(C.POINTER(C.c_double))


def sigma_error(sigma_hat, sigma_ref, ctx: Context | None = None) -> float:
    """Sum of |sigma_hat_i - sigma_ref_i|, the shorter list zero-padded (metrics.cpp:32-42)."""
    a = np.ascontiguousarray(sigma_hat, dtype=np.float64)
    b = np.ascontiguousarray(sigma_ref, dtype=np.float64)
    out = C.c_double()
    _check(lib().rk_sigma_error(_ctx(ctx), _pd(a), len(a), _pd(b), len(b), C.byref(out)))
    return out.value


def align_signs(u_hat, u_ref, sigma_ref=None, ctx: Context | None = None) -> np.ndarray:
    """Sign flips per column; with sigma_ref, Procrustes on degenerate clusters (metrics.cpp:44-93)."""
    h = np.ascontiguousarray(u_hat, dtype=np.float64)
    r = np.ascontiguousarray(u_ref, dtype=np.float64)
    if h.shape != r.shape:
        raise InvalidArgument("align_signs: shape mismatch")
    sg = np.ascontiguousarray(np.zeros(0) if sigma_ref is None else sigma_ref, dtype=np.float64)
    out = np.empty_like(h)
    _check(lib().rk_align_signs(_ctx(ctx), _pd(h), _pd(r), h.shape[0], h.shape[1], _pd(sg), len(sg), _pd(out)))
    return out


def left_vector_error(u_hat, u_ref, sigma_ref, ctx: Context | None = None) -> float:
    """Sum of |align_signs(u_hat) - u_ref| (metrics.cpp:95-103)."""
    h = np.ascontiguousarray(u_hat, dtype=np.float64)
    r = np.ascontiguousarray(u_ref, dtype=np.float64)
    if h.shape != r.shape:
        raise InvalidArgument("align_signs: shape mismatch")
    sg = np.ascontiguousarray(sigma_ref, dtype=np.float64)
    out = C.c_double()
    _check(lib().rk_left_vector_error(_ctx(ctx), _pd(h), _pd(r), h.shape[0], h.shape[1], _pd(sg), len(sg),
                                      C.byref(out)))
    return out.value


def numerical_rank(a, tol: float, ctx: Context | None = None) -> int:
    """Count of singular values above tol * sigma_max (metrics.cpp:105-114)."""
    d = np.ascontiguousarray(a, dtype=np.float64)
    out = C.c_uint64()
    _check(lib().rk_numerical_rank(_ctx(ctx), _pd(d), d.shape[0], d.shape[1], tol, C.byref(out)))
    return int(out.value)


def dev_left_vector_error(u_hat_t, u_ref_t, sigma_ref_t=None, ctx: Context | None = None) -> float:
    """left_vector_error on device tensors (torch, float64, row-major contiguous)."""
    out = C.c_double()
    ns = 0 if sigma_ref_t is None else int(sigma_ref_t.numel())
    _check(lib().rk_dev_left_vector_error(_ctx(ctx), C.c_void_p(u_hat_t.data_ptr()), C.c_void_p(u_ref_t.data_ptr()),
                                          u_hat_t.shape[0], u_hat_t.shape[1],
                                          C.c_void_p(sigma_ref_t.data_ptr() if ns else 0), ns, C.byref(out)))
    return out.value


def dev_sigma_error(a_t, b_t, ctx: Context | None = None) -> float:
    out = C.c_double()
    _check(lib().rk_dev_sigma_error(_ctx(ctx), C.c_void_p(a_t.data_ptr()), a_t.numel(), C.c_void_p(b_t.data_ptr()),
                                    b_t.numel(), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# records & pipeline

@dataclass
class BlockResultRecord:
    """proj/include/ranky/block_record.hpp:15-22 (payload rows x kept, row-major)"""
    block_index: int
    rows: int
    kept: int
    payload: np.ndarray

    def __eq__(self, o):
        return (self.block_index == o.block_index and self.rows == o.rows and self.kept == o.kept
                and np.array_equal(np.ravel(self.payload), np.ravel(o.payload)))


@dataclass
class BlockTask:
    """proj/include/ranky/pipeline.hpp:17-21"""
    block_index: int
    block: SparseMatrix
    keep: int = 0


def make_block_record(block_index: int, svd: SvdResult) -> BlockResultRecord:
    """proj/src/block_record.cpp:69-84"""
    if svd.u.shape[1] != len(svd.sigma):
        raise InvalidArgument("make_block_record: U columns do not match sigma")
    return BlockResultRecord(block_index, svd.u.shape[0], svd.u.shape[1], (svd.u * svd.sigma[None, :]).ravel())


def _records_of(r: _Records) -> list[BlockResultRecord]:
    """The records as views of the library's one payload buffer (no copy; the buffer
    lives as long as any record does)."""
    n = int(r.n_records)
    kept = _arr(r.kept, n, np.int64)
    offs = _arr(r.offset, n, np.int64)
    total = int(sum(kept)) * int(r.rows)
    flat = _take_array(r, "payload", total, (total,))
    return [BlockResultRecord(d, int(r.rows), int(kept[d]), flat[offs[d]:offs[d] + int(r.rows) * int(kept[d])])
            for d in range(n)]


def run_block_tasks(a: SparseMatrix, block_count: int, keep: int = 0, ctx: Context | None = None):
    """run_block_task for every block of partition_columns(a.cols, D) (GPU batch)"""
    v = a._view()
    out = _Records()
    L = lib()
    st = L.rk_run_block_tasks(_ctx(ctx), C.byref(v), block_count, keep, C.byref(out))
    try:
        _check(st)
        return _records_of(out)
    finally:
        L.rk_records_free(C.byref(out))


def run_block_task(task: BlockTask, ctx: Context | None = None) -> BlockResultRecord:
    """proj/src/pipeline.cpp:11-16"""
    rec = run_block_tasks(task.block, 1, task.keep, ctx)[0]
    rec.block_index = task.block_index
    return rec


def proxy_from_records(records, rows: int) -> ProxyMatrix:
    """proj/src/pipeline.cpp:18-59 (host container assembly)"""
    ordered = sorted(records, key=lambda r: r.block_index)
    for i in range(1, len(ordered)):
        if ordered[i - 1].block_index == ordered[i].block_index:
            raise InvalidArgument(f"duplicate block record index {ordered[i].block_index}")
    total = 0
    for r in ordered:
        if r.rows != rows:
            raise InvalidArgument(f"block record {r.block_index} has {r.rows} rows, expected {rows}")
        total += r.kept
    m = np.zeros((rows, total))
    offs, off = [], 0
    for r in ordered:
        offs.append(off)
        m[:, off:off + r.kept] = np.asarray(r.payload).reshape(rows, r.kept)
        off += r.kept
    offs.append(off)
    return ProxyMatrix(m, offs)


@dataclass
class PipelineResult:
    """proj/include/ranky/pipeline.hpp:30-36 (+ v when requested)"""
    svd: SvdResult
    report: RepairReport
    repaired: SparseMatrix | None
    partition: BlockPartition
    records: list
    timing: dict


def run_pipeline(a: SparseMatrix, block_count: int, method, keep: int = 0, seed: int = 0, workers: int = 1,
                 want_v: bool = False, top_k: int = 0, want_repaired: bool = True, want_records: bool = True,
                 ctx: Context | None = None) -> PipelineResult:
    """proj/src/pipeline.cpp:61-121 on the GPU. With want_v, svd.v = recover_right_vectors(
    repaired, U[:, :top_k], sigma[:top_k], kRankTol) -- the full Ranky SVD."""
    v = a._view()
    out = _Pipeline()
    flags = (WANT_V if want_v else 0) | (WANT_REPAIRED if want_repaired else 0) | (WANT_RECORDS if want_records else 0)
    L = lib()
    st = L.rk_run_pipeline(_ctx(ctx), C.byref(v), block_count, _method(method), keep, seed, workers, flags, top_k,
                           C.byref(out))
    try:
        _check(st)
        svd = _svd_of(out.svd)
        return PipelineResult(SvdResult(svd.u, svd.sigma, svd.v), _report_of(out.report),
                              _sparse_of(out.repaired) if want_repaired else None,
                              partition_columns(a.cols(), block_count),
                              _records_of(out.records) if want_records else [], out.timing.as_dict())
    finally:
        L.rk_pipeline_result_free(C.byref(out))


# ---------------------------------------------------------------------------
# device-resident path (bench / multi-GPU)

class DeviceMatrix:
    """A matrix uploaded once to HBM (rk_dev_matrix)."""

    def __init__(self, a: SparseMatrix, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self._a = a
        h = C.c_void_p()
        v = a._view()
        _check(lib().rk_dev_matrix_create(self.ctx.handle, C.byref(v), C.byref(h)))
        self.handle = h
        self.rows, self.cols, self.nnz = a.rows(), a.cols(), a.nnz()

    def close(self):
        if getattr(self, "handle", None):
            lib().rk_dev_matrix_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dev_full_svd(m: DeviceMatrix, block_count: int, method, keep: int = 0, seed: int = 0, want_v: bool = True,
                 top_k: int = 0):
    """repair -> blocks -> merge -> V on a device-resident matrix; returns (DevOutputs ptr, Timing)."""
    out = C.POINTER(DevOutputs)()
    t = Timing()
    _check(lib().rk_dev_full_svd(m.ctx.handle, m.handle, block_count, _method(method), keep, seed,
                                 WANT_V if want_v else 0, top_k, C.byref(out), C.byref(t)))
    return out, t


def dev_outputs_free(out):
    lib().rk_dev_outputs_free(out)


def dev_residual(m: DeviceMatrix, out) -> tuple[float, float]:
    """(||A - U diag(sigma) V^T||_F, ||A||_F) of device outputs, formed on the device
    (A = the repaired matrix the outputs reconstruct); test_support.hpp:57-70."""
    r, a = C.c_double(), C.c_double()
    _check(lib().rk_dev_residual(m.ctx.handle, m.handle, out, C.byref(r), C.byref(a)))
    return r.value, a.value


class _CudaArray:
    """__cuda_array_interface__ over library-owned device memory (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def dev_outputs_tensors(out):
    """(sigma, U, V) of rk_dev_outputs as torch views of the library's HBM buffers
    (valid until dev_outputs_free); V is None without RK_WANT_V."""
    import torch
    o = out.contents
    dev = torch.device("cuda", torch.cuda.current_device())
    sig = torch.as_tensor(_CudaArray(o.d_sigma, (o.k_sigma,)), device=dev) if o.k_sigma else None
    u = torch.as_tensor(_CudaArray(o.d_u, (o.rows, o.k_sigma)), device=dev) if o.k_sigma else None
    v = torch.as_tensor(_CudaArray(o.d_v, (o.cols, o.k_v)), device=dev) if o.d_v else None
    return sig, u, v


# ---------------------------------------------------------------------------
# RNKY block records (proj/src/block_record.cpp:51-144)

def crc32(data) -> int:
    """block_record.cpp:53-68 (CRC-32, reflected 0xEDB88320)"""
    b = bytes(data) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data).tobytes()
    return int(lib().rk_crc32(b, len(b)))


def write_block_record(record: BlockResultRecord, path) -> None:
    """block_record.cpp:86-106: byte-identical RNKY file"""
    pay = np.ascontiguousarray(record.payload, dtype=np.float64).ravel()
    if pay.size != record.rows * record.kept:
        raise InvalidArgument("block record payload size mismatch")
    _check(lib().rk_write_block_record(record.block_index, record.rows, record.kept,
                                       pay.ctypes.data_as(C.POINTER(C.c_double)), os.fsencode(str(path))))


def read_block_record(path) -> BlockResultRecord:
    """block_record.cpp:108-144 (RecordError on damage)"""
    idx, rows, kept = C.c_uint32(), C.c_uint32(), C.c_uint32()
    p = C.POINTER(C.c_double)()
    _check(lib().rk_read_block_record(os.fsencode(str(path)), C.byref(idx), C.byref(rows), C.byref(kept), C.byref(p)))
    n = rows.value * kept.value
    try:
        pay = np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0)
    finally:
        lib().rk_host_free(p)
    return BlockResultRecord(idx.value, rows.value, kept.value, pay)


def write_records(records, path_prefix, ctx: Context | None = None) -> None:
    """every record to '<path_prefix><block index>.rnky' (payload CRCs on the GPU);
    records must be those of one pipeline call (block_index = 0, 1, ...)"""
    if not records:
        return
    rows = records[0].rows
    kept = np.array([r.kept for r in records], dtype=np.uint32)
    offset = np.zeros(len(records), dtype=np.uint64)
    offset[1:] = np.cumsum(kept.astype(np.uint64) * rows)[:-1]
    payload = np.ascontiguousarray(np.concatenate([np.asarray(r.payload, np.float64).ravel() for r in records]))
    if any(r.block_index != d or r.rows != rows for d, r in enumerate(records)):
        raise InvalidArgument("write_records: records must be blocks 0..n-1 of one matrix")
    rec = _Records(len(records), rows, kept.ctypes.data_as(C.POINTER(C.c_uint32)),
                   offset.ctypes.data_as(C.POINTER(C.c_uint64)), payload.ctypes.data_as(C.POINTER(C.c_double)))
    _check(lib().rk_write_records(_ctx(ctx), C.byref(rec), os.fsencode(str(path_prefix))))


# ---------------------------------------------------------------------------
# library-owned multi-GPU runs (rk_multi_*, rk_dist_*, rk_dev_sharded_full_svd)

class Multi:
    """Several devices driven from this process (rk_multi_*). `devices` may repeat a
    device (its shards then share it) -- e.g. [0, 0] runs the two-shard protocol on
    one GPU, bitwise the same as two processes on two GPUs."""

    def __init__(self, devices):
        d = (C.c_int32 * len(devices))(*devices)
        self.handle = C.c_void_p()
        _check(lib().rk_multi_create(d, len(devices), C.byref(self.handle)))
        self.devices = list(devices)

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            lib().rk_multi_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_pipeline(self, a: SparseMatrix, block_count: int, method, keep: int = 0, seed: int = 0,
                     want_v: bool = False, top_k: int = 0, want_repaired: bool = True,
                     want_records: bool = True) -> PipelineResult:
        """run_pipeline (proj/src/pipeline.cpp:61-121) over all the devices."""
        v = a._view()
        out = _Pipeline()
        flags = (WANT_V if want_v else 0) | (WANT_REPAIRED if want_repaired else 0) | \
            (WANT_RECORDS if want_records else 0)
        L = lib()
        st = L.rk_multi_run_pipeline(self.handle, C.byref(v), block_count, _method(method), keep, seed, flags, top_k,
                                     C.byref(out))
        try:
            _check(st)
            svd = _svd_of(out.svd)
            return PipelineResult(SvdResult(svd.u, svd.sigma, svd.v), _report_of(out.report),
                                  _sparse_of(out.repaired) if want_repaired else None,
                                  partition_columns(a.cols(), block_count),
                                  _records_of(out.records) if want_records else [], out.timing.as_dict())
        finally:
            L.rk_pipeline_result_free(C.byref(out))


def dev_sharded_full_svd(m: DeviceMatrix, block_count: int, method, keep: int, seed: int, world: int, rank: int,
                         allgather, want_v: bool = True, top_k: int = 0):
    """One rank's share of the library-orchestrated sharded run with the caller's
    all-gather: allgather(mine, all) gets torch float64 CUDA tensors (count and
    world*count doubles) and must fill `all` in rank order before returning.
    Returns (DevOutputs ptr, Timing, col_lo, col_hi)."""
    import torch

    def cb(user, d_mine, d_all, count):
        mine = torch.as_tensor(_CudaArray(d_mine, (count,)), device="cuda")
        alls = torch.as_tensor(_CudaArray(d_all, (count * world,)), device="cuda")
        allgather(mine, alls)
        # the C ABI's contract: `all` is filled when the callback returns. torch's collectives and
        # copies are asynchronous on torch's current stream, which is not the library's (a context
        # on torch's default stream runs on its own non-blocking stream), so wait for them here
        torch.cuda.current_stream().synchronize()

    fn = ALLGATHER_FN(cb)
    out = C.POINTER(DevOutputs)()
    t = Timing()
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib().rk_dev_sharded_full_svd(m.ctx.handle, m.handle, block_count, _method(method), keep, seed,
                                         WANT_V if want_v else 0, top_k, world, rank, fn, None, C.byref(out),
                                         C.byref(t), C.byref(lo), C.byref(hi)))
    return out, t, lo.value, hi.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().rk_nccl_unique_id(buf))
    return bytes(buf)


class Dist:
    """One process per GPU with the library's own NCCL communicator (rk_dist_*)."""

    def __init__(self, ctx: Context, world: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * 128)(*uid)
        self.handle = C.c_void_p()
        _check(lib().rk_dist_create(ctx.handle, world, rank, buf, C.byref(self.handle)))

    def full_svd(self, m: DeviceMatrix, block_count: int, method, keep: int = 0, seed: int = 0, want_v: bool = True,
                 top_k: int = 0):
        out = C.POINTER(DevOutputs)()
        t = Timing()
        lo, hi = C.c_uint64(), C.c_uint64()
        _check(lib().rk_dist_full_svd(self.handle, m.handle, block_count, _method(method), keep, seed,
                                      WANT_V if want_v else 0, top_k, C.byref(out), C.byref(t), C.byref(lo),
                                      C.byref(hi)))
        return out, t, lo.value, hi.value

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            lib().rk_dist_destroy(self.handle)
            self.handle = C.c_void_p()
