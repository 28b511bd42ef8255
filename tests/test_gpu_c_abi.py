"""The C ABI from plain C (tests/c/c_abi_smoke.c compiled with gcc against
include/ranky_b200.h and libranky_b200.so): the boundary a cgo / JNI / N-API
binding sees, with no Python or C++ in between."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_against_the_abi(tmp_path):
    exe = tmp_path / "c_abi_smoke"
    lib = os.path.join(ROOT, "paper_2009_09767_b200")
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "c_abi_smoke.c"), "-o", str(exe), "-L", lib, "-lranky_b200",
                    f"-Wl,-rpath,{lib}", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c abi smoke:" in r.stdout
