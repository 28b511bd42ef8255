"""The five BASELINE.json workloads, generated deterministically by csrc/gen.c.

Public datasets are not involved: the paper's data is proprietary and the
BASELINE configs are synthetic by definition. Each generator is seeded exactly
as BASELINE.json states; DESIGN.md documents the interpretation of each line.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from .ranky import ENTRY_DTYPE, SparseMatrix

_PKG = os.path.dirname(os.path.abspath(__file__))
GEN_SO = os.path.join(_PKG, "libranky_gen.so")
GEN_SRC = os.path.join(_PKG, "csrc", "gen.c")

VAL_ONE, VAL_UNIFORM_PM1, VAL_NORMAL, VAL_UNIFORM_01 = 0, 1, 2, 3


def build_gen() -> str:
    if not os.path.exists(GEN_SO) or os.path.getmtime(GEN_SO) < os.path.getmtime(GEN_SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", GEN_SO, GEN_SRC, "-lm"], check=True)
    return GEN_SO


_gen = None


def _lib():
    global _gen
    if _gen is None:
        L = C.CDLL(build_gen())
        u64, dbl, i32 = C.c_uint64, C.c_double, C.c_int
        L.rkg_uniform.argtypes = [u64, u64, dbl, i32, u64, u64, u64, u64, C.POINTER(u64)]
        L.rkg_uniform.restype = C.c_void_p
        L.rkg_zipf.argtypes = [u64, u64, dbl, dbl, i32, u64, C.POINTER(u64)]
        L.rkg_zipf.restype = C.c_void_p
        L.rkg_zipf_mean.argtypes = [u64, dbl]
        L.rkg_zipf_mean.restype = dbl
        L.rkg_synth_bipartite.argtypes = [u64, u64, dbl, u64, C.POINTER(u64)]
        L.rkg_synth_bipartite.restype = C.c_void_p
        L.rkg_planted.argtypes = [u64, u64, dbl, u64, dbl, dbl, u64, C.POINTER(u64)]
        L.rkg_planted.restype = C.c_void_p
        L.rkg_free.argtypes = [C.c_void_p]
        _gen = L
    return _gen


def _take(ptr, n) -> np.ndarray:
    L = _lib()
    if n == 0:
        L.rkg_free(ptr)
        return np.zeros(0, dtype=ENTRY_DTYPE)
    buf = (C.c_char * (n * ENTRY_DTYPE.itemsize)).from_address(ptr)
    e = np.frombuffer(buf, dtype=ENTRY_DTYPE).copy()
    L.rkg_free(ptr)
    return e


def uniform(rows, cols, density, kind, seed, D=0, plant_blocks=0, plant_rows=0) -> SparseMatrix:
    n = C.c_uint64()
    p = _lib().rkg_uniform(rows, cols, density, kind, seed, D, plant_blocks, plant_rows, C.byref(n))
    if not p:
        raise MemoryError("generator allocation failed")
    return SparseMatrix._trusted(rows, cols, _take(p, n.value))


def zipf(rows, cols, mean_degree, s, kind, seed) -> SparseMatrix:
    L = _lib()
    p_nonempty = min(1.0, mean_degree / L.rkg_zipf_mean(rows, s))
    n = C.c_uint64()
    p = L.rkg_zipf(rows, cols, p_nonempty, s, kind, seed, C.byref(n))
    return SparseMatrix._trusted(rows, cols, _take(p, n.value))


def synth_bipartite(rows, cols, density, seed) -> SparseMatrix:
    """proj/src/synth.cpp:14-29 restated (Bernoulli cells of value 1.0)."""
    n = C.c_uint64()
    p = _lib().rkg_synth_bipartite(rows, cols, density, seed, C.byref(n))
    return SparseMatrix._trusted(rows, cols, _take(p, n.value))


def planted(rows, cols, density, k, decay, noise, seed) -> SparseMatrix:
    """c5's planted spectrum: mask(density) o (P diag(decay^j) Q^T) + noise N(0,1) on
    the nonzeros, P (rows x k) and Q (cols x k) orthonormal from seeded Gaussians."""
    n = C.c_uint64()
    p = _lib().rkg_planted(rows, cols, density, k, decay, noise, seed, C.byref(n))
    if not p:
        raise MemoryError("planted generator failed")
    return SparseMatrix._trusted(rows, cols, _take(p, n.value))


@dataclass(frozen=True)
class Config:
    name: str
    rows: int
    cols: int
    blocks: int
    method: str
    seed: int
    keep: int
    top_k: int
    description: str

    def generate(self, scale_cols: int | None = None) -> SparseMatrix:
        """The matrix; scale_cols (a multiple of `blocks`) shrinks N for quick tests."""
        n = scale_cols or self.cols
        if self.name == "c1":
            return uniform(self.rows, n, 0.01, VAL_UNIFORM_PM1, self.seed, self.blocks, 4, 8)
        if self.name == "c2":
            return uniform(self.rows, n, 0.005, VAL_NORMAL, self.seed, self.blocks, round(0.1 * self.blocks), 16)
        if self.name == "c3":
            return zipf(self.rows, n, 0.002 * self.rows, 1.1, VAL_UNIFORM_01, self.seed)
        if self.name == "c4":
            return uniform(self.rows, n, 0.001, VAL_NORMAL, self.seed)
        if self.name == "c5":
            return planted(self.rows, n, 0.0005, 64, 0.9, 1e-6, self.seed)
        raise ValueError(f"unknown config {self.name}")


CONFIGS = {
    "c1": Config("c1", 64, 8192, 16, "random", 0, 0, 0,
                 "M=64 N=8192 1% uniform U(-1,1) seed 0, 16 blocks, 8 rows zeroed in 4 blocks, RandomChecker"),
    "c2": Config("c2", 256, 262144, 64, "random", 1, 0, 0,
                 "M=256 N=262144 0.5% uniform N(0,1) seed 1, 64 blocks, 16 empty rows planted in 6 blocks, "
                 "RandomChecker"),
    "c3": Config("c3", 512, 4194304, 512, "neighbor", 2, 0, 0,
                 "M=512 N=4194304 Zipf(1.1) column degrees (mean 1.024/col) U(0,1) seed 2, 512 blocks, "
                 "NeighborChecker"),
    "c4": Config("c4", 1024, 16777216, 1024, "neighbor-random", 3, 0, 0,
                 "M=1024 N=16777216 0.1% uniform N(0,1) seed 3, 1024 blocks, NeighborRandomChecker"),
    "c5": Config("c5", 2048, 67108864, 4096, "neighbor-random", 4, 64, 64,
                 "planted spectrum M=2048 N=67108864: mask(0.05% uniform, seed 4) o (P diag(0.9^k) Q^T) + 1e-6 N(0,1), "
                 "P, Q orthonormal (k=64) from seeded Gaussians; 4096 blocks, NeighborRandomChecker, keep 64, top-64"),
}
