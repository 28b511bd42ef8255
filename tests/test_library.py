"""The C-ABI library: it loads, it exports every entry point include/ranky_b200.h
declares, it was built for sm_100a, and without a CUDA device the product path
raises instead of falling back to the CPU. No compute calls here."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ranky_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^RK_API\s+[\w\s\*]+?\b(rk_\w+)\(", src, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("rk_repair", "rk_block_svd", "rk_dense_svd", "rk_proxy_svd", "rk_recover_right_vectors",
                 "rk_run_pipeline", "rk_find_lonely_rows", "rk_dev_full_svd", "rk_dev_shard_factor"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2009_09767_b200 import ranky
    lib = ctypes.CDLL(ranky.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert ranky.lib().rk_abi_version() == 1


def test_library_is_sm100a():
    from paper_2009_09767_b200 import ranky
    out = subprocess.run(["cuobjdump", "--list-elf", ranky.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import numpy as np
    import paper_2009_09767_b200 as rk
    with pytest.raises(rk.ranky.CudaError):
        rk.dense_svd(np.eye(3))
