"""In-tree build of libranky_b200.so (sm_100a) with nvcc.

The shared library is the product: the CUDA kernels plus the C ABI declared in
include/ranky_b200.h. It is built in place so that it travels with the repo
snapshot to the GPU box (a JIT cache would not).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libranky_b200.so")
SOURCES = ["rk_scan.cu", "rk_ingest.cu", "rk_repair.cu", "rk_compact.cu", "rk_dense.cu", "rk_metrics.cu", "rk_eval.cu", "rk_workspace.cu", "rk_mm.cu", "rk_eig.cu", "rk_records.cu", "rk_qr.cu", "rk_gram.cu", "rk_precond.cu", "rk_spmm.cu",
           "rk_pipeline.cu", "rk_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _needs(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "ranky_b200.h"))
    cc = nvcc()
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _needs(o, [s] + headers):
            exp = ["-DRK_EXPERIMENTS"] if os.environ.get("RK_EXPERIMENTS") == "1" else []
            cmd = [cc, *ARCH, *FLAGS, *exp, *os.environ.get("RK_NVCC_EXTRA", "").split(), "-I", os.path.join(ROOT, "include"),
                   "-I", CSRC, "-c", s, "-o", o]
            jobs.append(cmd)
    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stderr, r.stdout, file=sys.stderr)
        return r
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _needs(LIB, objs):
        cmd = [cc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl",
               "-lpthread"]
        run(cmd)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
