"""oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front end over the two CPU oracles of the Ranky hot path:

* ``kind="port"``      -- the C restatement ``oracle/ranky_oracle.c``
  (built into ``oracle/_build/libranky_oracle.so``), and
* ``kind="reference"`` -- the unmodified reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` into
  ``oracle/_ref/libranky_ref.so`` (wrapped by ``oracle/ref_capi.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg import this module. The CUDA product path never does.

Sparse matrices are passed as sorted COO triples ``(rows, cols, r, c, v)``
with ``r, c`` uint64 and ``v`` float64, exactly the entry order of the
reference ``SparseMatrix`` (proj/src/sparse_matrix.cpp:9-34).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libranky_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libranky_ref.so")
REF_ACCEPTANCE = os.path.join(HERE, "_ref", "ranky_acceptance")

METHODS = {"random": 0, "neighbor": 1, "neighbor-random": 2, "none": 3}


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str, residual: float = 0.0):
        super().__init__(message)
        self.code = code
        self.residual = residual


class _Res(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("message", C.c_char * 512), ("residual", C.c_double),
        ("n_edges", C.c_uint64), ("e_block", C.POINTER(C.c_uint64)), ("e_row", C.POINTER(C.c_uint64)),
        ("e_col", C.POINTER(C.c_uint64)), ("e_mech", C.POINTER(C.c_int32)),
        ("n_blocks", C.c_uint64), ("lonely", C.POINTER(C.c_uint64)), ("fallback", C.c_uint64),
        ("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
        ("r", C.POINTER(C.c_uint64)), ("c", C.POINTER(C.c_uint64)), ("v", C.POINTER(C.c_double)),
        ("u_rows", C.c_uint64), ("u_cols", C.c_uint64), ("u", C.POINTER(C.c_double)),
        ("n_sigma", C.c_uint64), ("sigma", C.POINTER(C.c_double)),
        ("has_v", C.c_int), ("v_rows", C.c_uint64), ("v_cols", C.c_uint64), ("vm", C.POINTER(C.c_double)),
        ("n_records", C.c_uint64), ("rec_kept", C.POINTER(C.c_uint32)), ("rec_payload", C.POINTER(C.c_double)),
        ("t_repair", C.c_double), ("t_blocks", C.c_double), ("t_proxy", C.c_double),
    ]


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True)


@dataclass
class Result:
    edges: np.ndarray | None = None      # (E, 4): block, row, col, mechanism(0 random / 1 neighbor)
    lonely_counts: np.ndarray | None = None
    fallback_count: int = 0
    matrix: tuple | None = None           # (rows, cols, r, c, v)
    u: np.ndarray | None = None
    sigma: np.ndarray | None = None
    v: np.ndarray | None = None
    records: list = field(default_factory=list)  # list of (rows, kept) payload arrays
    times: tuple = (0.0, 0.0, 0.0)

    def to_log(self) -> str:
        """RepairReport::to_log -- proj/src/repair.cpp:27-40."""
        names = {0: "random", 1: "neighbor"}
        out = [f"{b}\t{r}\t{c}\t{names[int(m)]}\n" for b, r, c, m in self.edges]
        out.append("# lonely=" + ",".join(str(int(x)) for x in self.lonely_counts)
                   + f" fallback={self.fallback_count}\n")
        return "".join(out)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        p = "or_" if kind == "port" else "ref_"
        self.p = p
        L = self.lib
        u64, dbl, i32 = C.c_uint64, C.c_double, C.c_int
        pu64, pdbl = C.POINTER(C.c_uint64), C.POINTER(C.c_double)
        R = C.POINTER(_Res)
        self._free = getattr(L, p + "free")
        self._free.argtypes = [R]
        fn = getattr(L, p + "repair"); fn.argtypes = [u64, u64, u64, pu64, pu64, pdbl, u64, i32, u64]; fn.restype = R
        fn = getattr(L, p + "dense_svd"); fn.argtypes = [u64, u64, pdbl]; fn.restype = R
        fn = getattr(L, p + "block_svd"); fn.argtypes = [u64, u64, u64, pu64, pu64, pdbl, u64]; fn.restype = R
        fn = getattr(L, p + "recover_right_vectors")
        fn.argtypes = [u64, u64, u64, pu64, pu64, pdbl, pdbl, u64, u64, pdbl, u64, dbl]; fn.restype = R
        fn = getattr(L, p + "run_pipeline")
        fn.argtypes = [u64, u64, u64, pu64, pu64, pdbl, u64, i32, u64, u64, u64]; fn.restype = R
        fn = getattr(L, p + "rng_stream"); fn.argtypes = [u64, u64, u64, u64, pu64]; fn.restype = None
        fn = getattr(L, p + "rng_below"); fn.argtypes = [u64, u64, u64, u64]; fn.restype = u64
        fn = getattr(L, p + "find_lonely_rows"); fn.argtypes = [u64, u64, u64, pu64, pu64, u64, u64, pu64]; fn.restype = u64
        if kind == "reference":
            fn = L.ref_full_svd
            fn.argtypes = [u64, u64, u64, pu64, pu64, pdbl, u64, i32, u64, u64, u64, u64]; fn.restype = R
            fn = L.ref_proxy_svd_records
            fn.argtypes = [u64, u64, C.POINTER(C.c_uint32), pdbl]; fn.restype = R
            fn = L.ref_synth_bipartite; fn.argtypes = [u64, u64, dbl, u64]; fn.restype = R
        else:
            fn = L.or_synth_bipartite; fn.argtypes = [u64, u64, dbl, u64, pu64, pu64, pdbl]; fn.restype = u64

    # -- helpers ---------------------------------------------------------
    @staticmethod
    def _coo(a):
        rows, cols, r, c, v = a
        r = np.ascontiguousarray(r, dtype=np.uint64)
        c = np.ascontiguousarray(c, dtype=np.uint64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        return rows, cols, r, c, v

    @staticmethod
    def _p(x, t):
        return x.ctypes.data_as(C.POINTER(t))

    def _take(self, rp) -> Result:
        res = rp.contents
        try:
            if res.status != 0:
                raise OracleError(res.status, res.message.decode(), res.residual)
            out = Result()
            if res.n_blocks or res.n_edges:
                e = np.zeros((res.n_edges, 4), dtype=np.int64)
                e[:, 0] = _arr(res.e_block, res.n_edges, np.int64)
                e[:, 1] = _arr(res.e_row, res.n_edges, np.int64)
                e[:, 2] = _arr(res.e_col, res.n_edges, np.int64)
                e[:, 3] = _arr(res.e_mech, res.n_edges, np.int64)
                out.edges = e
                out.lonely_counts = _arr(res.lonely, res.n_blocks, np.int64)
                out.fallback_count = int(res.fallback)
            if res.r:
                out.matrix = (int(res.rows), int(res.cols), _arr(res.r, res.nnz, np.uint64),
                              _arr(res.c, res.nnz, np.uint64), _arr(res.v, res.nnz, np.float64))
            if res.u or res.u_rows:
                out.u = _arr(res.u, res.u_rows * res.u_cols, np.float64).reshape(int(res.u_rows), int(res.u_cols))
            if res.sigma or res.n_sigma == 0:
                out.sigma = _arr(res.sigma, res.n_sigma, np.float64)
            if res.has_v:
                out.v = _arr(res.vm, res.v_rows * res.v_cols, np.float64).reshape(int(res.v_rows), int(res.v_cols))
            if res.n_records:
                kept = _arr(res.rec_kept, res.n_records, np.int64)
                rows = int(res.u_rows)
                total = int(sum(kept)) * rows
                flat = _arr(res.rec_payload, total, np.float64)
                off = 0
                for k in kept:
                    out.records.append(flat[off:off + rows * k].reshape(rows, int(k)))
                    off += rows * int(k)
            out.times = (res.t_repair, res.t_blocks, res.t_proxy)
            return out
        finally:
            self._free(rp)

    # -- API (names follow proj/include/ranky) ---------------------------
    def rng_stream(self, seed, block, row, n):
        out = np.zeros(n, dtype=np.uint64)
        getattr(self.lib, self.p + "rng_stream")(seed, block, row, n, self._p(out, C.c_uint64))
        return out

    def rng_below(self, seed, block, row, bound):
        return int(getattr(self.lib, self.p + "rng_below")(seed, block, row, bound))

    def synth_bipartite(self, rows, cols, density, seed):
        if self.kind == "reference":
            m = self._take(self.lib.ref_synth_bipartite(rows, cols, density, seed)).matrix
            return m
        n = self.lib.or_synth_bipartite(rows, cols, density, seed, None, None, None)
        r = np.zeros(n, np.uint64); c = np.zeros(n, np.uint64); v = np.zeros(n, np.float64)
        self.lib.or_synth_bipartite(rows, cols, density, seed, self._p(r, C.c_uint64),
                                    self._p(c, C.c_uint64), self._p(v, C.c_double))
        return (rows, cols, r, c, v)

    def find_lonely_rows(self, a, D, d):
        rows, cols, r, c, v = self._coo(a)
        out = np.zeros(max(rows, 1), dtype=np.uint64)
        n = getattr(self.lib, self.p + "find_lonely_rows")(rows, cols, len(r), self._p(r, C.c_uint64),
                                                         self._p(c, C.c_uint64), D, d, self._p(out, C.c_uint64))
        return out[:n].astype(np.int64)

    def repair(self, a, D, method, seed) -> Result:
        rows, cols, r, c, v = self._coo(a)
        return self._take(getattr(self.lib, self.p + "repair")(
            rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double),
            D, METHODS[method], seed))

    def dense_svd(self, a: np.ndarray) -> Result:
        a = np.ascontiguousarray(a, dtype=np.float64)
        return self._take(getattr(self.lib, self.p + "dense_svd")(a.shape[0], a.shape[1], self._p(a, C.c_double)))

    def block_svd(self, a, keep) -> Result:
        rows, cols, r, c, v = self._coo(a)
        return self._take(getattr(self.lib, self.p + "block_svd")(
            rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double), keep))

    def recover_right_vectors(self, a, u, sigma, tol=1e-10) -> np.ndarray:
        rows, cols, r, c, v = self._coo(a)
        u = np.ascontiguousarray(u, dtype=np.float64)
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        res = self._take(getattr(self.lib, self.p + "recover_right_vectors")(
            rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double),
            self._p(u, C.c_double), u.shape[0], u.shape[1], self._p(s, C.c_double), len(s), tol))
        return res.v

    def run_pipeline(self, a, D, method, keep=0, seed=0, workers=1) -> Result:
        rows, cols, r, c, v = self._coo(a)
        return self._take(getattr(self.lib, self.p + "run_pipeline")(
            rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double),
            D, METHODS[method], keep, seed, workers))

    def full_svd(self, a, D, method, keep=0, seed=0, workers=1, top_k=0) -> Result:
        """run_pipeline + recover_right_vectors (reference only)."""
        rows, cols, r, c, v = self._coo(a)
        return self._take(self.lib.ref_full_svd(
            rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double),
            D, METHODS[method], keep, seed, workers, top_k))

    def proxy_svd_records(self, records) -> Result:
        """proxy_from_records + proxy_svd (reference only)."""
        rows = records[0].shape[0]
        kept = np.array([rec.shape[1] for rec in records], dtype=np.uint32)
        flat = np.ascontiguousarray(np.concatenate([rec.ravel() for rec in records]), dtype=np.float64)
        return self._take(self.lib.ref_proxy_svd_records(rows, len(records), self._p(kept, C.c_uint32),
                                                         self._p(flat, C.c_double)))


    # ---- Matrix Market (reference only): proj/src/matrix_market.cpp:38-132 ----
    def load_matrix_market(self, path):
        """-> (rows, cols, r, c, v); raises OracleError(6, "... (line L)", residual=L) on ParseError"""
        fn = self.lib.ref_load_matrix_market
        fn.restype = C.POINTER(_Res)
        fn.argtypes = [C.c_char_p]
        return self._take(fn(str(path).encode())).matrix

    def save_matrix_market(self, a, path):
        """The reference's writer in its own process (oracle/_ref/ref_mm_save): inside a
        Python process that has loaded numpy's bundled libraries its std::to_chars(double)
        path crashes under ctypes."""
        import subprocess
        import tempfile
        rows, cols, r, c, v = self._coo(a)
        exe = os.path.join(os.path.dirname(REF_SO), "ref_mm_save")
        with tempfile.NamedTemporaryFile(suffix=".coo", delete=False) as f:
            f.write(np.array([rows, cols, len(r)], dtype=np.uint64).tobytes())
            f.write(r.tobytes()); f.write(c.tobytes()); f.write(v.tobytes())
            tmp = f.name
        try:
            if subprocess.run([exe, tmp, str(path)]).returncode:
                raise OracleError(4, "save_matrix_market failed")
        finally:
            os.unlink(tmp)

    # ---- evaluation metrics (reference only): proj/src/metrics.cpp:32-114 ----
    def sigma_error(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64); b = np.ascontiguousarray(b, dtype=np.float64)
        fn = self.lib.ref_sigma_error
        fn.restype = C.c_double
        fn.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_double), C.c_uint64]
        return float(fn(self._p(a, C.c_double), len(a), self._p(b, C.c_double), len(b)))

    def align_signs(self, u_hat, u_ref, sigma=None) -> np.ndarray:
        h = np.ascontiguousarray(u_hat, dtype=np.float64); r = np.ascontiguousarray(u_ref, dtype=np.float64)
        s = np.ascontiguousarray(np.zeros(0) if sigma is None else sigma, dtype=np.float64)
        out = np.zeros_like(h)
        fn = self.lib.ref_align_signs
        fn.restype = C.c_int
        pd = C.POINTER(C.c_double)
        fn.argtypes = [pd, pd, C.c_uint64, C.c_uint64, pd, C.c_uint64, pd]
        if fn(self._p(h, C.c_double), self._p(r, C.c_double), h.shape[0], h.shape[1], self._p(s, C.c_double),
              len(s), self._p(out, C.c_double)):
            raise OracleError(1, "align_signs: invalid argument")
        return out

    def left_vector_error(self, u_hat, u_ref, sigma=None) -> float:
        h = np.ascontiguousarray(u_hat, dtype=np.float64); r = np.ascontiguousarray(u_ref, dtype=np.float64)
        s = np.ascontiguousarray(np.zeros(0) if sigma is None else sigma, dtype=np.float64)
        fn = self.lib.ref_left_vector_error
        fn.restype = C.c_double
        pd = C.POINTER(C.c_double)
        fn.argtypes = [pd, pd, C.c_uint64, C.c_uint64, pd, C.c_uint64]
        return float(fn(self._p(h, C.c_double), self._p(r, C.c_double), h.shape[0], h.shape[1],
                        self._p(s, C.c_double), len(s)))

    def numerical_rank(self, a, tol) -> int:
        a = np.ascontiguousarray(a, dtype=np.float64)
        fn = self.lib.ref_numerical_rank
        fn.restype = C.c_uint64
        fn.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_uint64, C.c_double]
        return int(fn(self._p(a, C.c_double), a.shape[0], a.shape[1], tol))

    def sampled_pipeline(self, a, D, method, keep, seed, workers, sample, slice_cols, phase) -> np.ndarray:
        """ref_sampled_pipeline (reference only): per-stage std::chrono times of the
        reference's run_pipeline stages on a block sample (see ref_capi.cpp)."""
        rows, cols, r, c, v = self._coo(a)
        fn = self.lib.ref_sampled_pipeline
        fn.restype = C.c_int
        fn.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                       C.POINTER(C.c_double), C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                       C.POINTER(C.c_uint64), C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_double)]
        smp = np.ascontiguousarray(sample, dtype=np.uint64)
        t = np.zeros(8)
        st = fn(rows, cols, len(r), self._p(r, C.c_uint64), self._p(c, C.c_uint64), self._p(v, C.c_double), D,
                METHODS[method], keep, seed, workers, self._p(smp, C.c_uint64), len(smp), slice_cols, phase,
                self._p(t, C.c_double))
        if st:
            raise OracleError(4, f"ref_sampled_pipeline failed ({st})")
        return t

    # ---- RNKY records (reference only): block_record.cpp:53-144 ----
    def crc32(self, data: bytes) -> int:
        self.lib.ref_crc32.restype = C.c_uint32
        self.lib.ref_crc32.argtypes = [C.c_char_p, C.c_uint64]
        return int(self.lib.ref_crc32(data, len(data)))

    def write_block_record(self, index, payload, path):
        p = np.ascontiguousarray(payload, dtype=np.float64)
        self.lib.ref_write_block_record.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double),
                                                    C.c_char_p]
        if self.lib.ref_write_block_record(index, p.shape[0], p.shape[1], self._p(p, C.c_double), str(path).encode()):
            raise OracleError(4, "write_block_record failed")

    def read_block_record(self, path, cap=1 << 24):
        """-> (index, payload) ; raises OracleError(7) on the reference's RecordError"""
        idx, rows, kept = C.c_uint32(), C.c_uint32(), C.c_uint32()
        out = np.zeros(cap, dtype=np.float64)
        self.lib.ref_read_block_record.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                                   C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_uint64]
        st = self.lib.ref_read_block_record(str(path).encode(), C.byref(idx), C.byref(rows), C.byref(kept),
                                            self._p(out, C.c_double), cap)
        if st == 1:
            raise OracleError(7, "RecordError")
        if st:
            raise OracleError(4, "read_block_record failed")
        return idx.value, out[:rows.value * kept.value].reshape(rows.value, kept.value).copy()


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)
