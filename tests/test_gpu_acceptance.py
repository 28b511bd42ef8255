"""The reference's own acceptance suite (proj/tests/acceptance_main.cpp), relinked
with its hot-path objects (repair, svd, proxy, pipeline) replaced by the B200
drop-in (paper_2009_09767_b200/dropin/ranky_dropin.cpp -> libranky_b200.so).
The binary is built by oracle/Makefile (target dropin) where the reference
sources exist and travels prebuilt in oracle/_ref."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ranky_acceptance_b200")

pytestmark = pytest.mark.gpu


def test_reference_acceptance_suite_on_b200_dropin():
    if not os.path.exists(BIN):
        pytest.skip("relinked acceptance binary not built (needs the reference sources)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    text = out.stdout + out.stderr
    print(text)
    passed = [l for l in text.splitlines() if l.startswith("PASS")]
    failed = [l for l in text.splitlines() if l.startswith("FAIL")]
    assert not failed, failed
    assert len(passed) == 8, text
    assert out.returncode == 0


def test_reference_workspace_tests_on_b200_dropin():
    """proj/tests/repair_test.cpp's RepairWorkspace cases (tests/c/workspace_dropin_test.cpp)
    through the drop-in's RepairWorkspace (rk_workspace_* device workspace)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ranky_workspace_b200")
    if not os.path.exists(exe):
        pytest.skip("workspace drop-in test not built (needs the reference sources)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout + out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


def test_reference_acceptance_suite_on_two_shards():
    """The same suite with RANKY_DEVICES=0,0: the drop-in's run_pipeline shards the
    blocks over two device contexts (rk_multi_run_pipeline: concurrent shards, the
    factor exchange by device copies, the shared tree top)."""
    if not os.path.exists(BIN):
        pytest.skip("relinked acceptance binary not built (needs the reference sources)")
    env = dict(os.environ, RANKY_DEVICES="0,0")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env=env)
    text = out.stdout + out.stderr
    print(text)
    assert not [l for l in text.splitlines() if l.startswith("FAIL")], text
    assert len([l for l in text.splitlines() if l.startswith("PASS")]) == 8, text
    assert out.returncode == 0
