"""Drop-in check: the reference's OWN allocator/simulator/acceptance tests pass with its
KVCacheManager replaced by paper_2405_04437_b200.KVCacheManager (C++ core, shadow backend).
Build container only (needs /root/reference)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import REF_SRC, ROOT

REF_TESTS = REF_SRC.parent / "tests"


@pytest.mark.reference
@pytest.mark.parametrize("module,select", [
    ("test_manager.py", None),
    ("test_simulator.py", None),
    ("test_acceptance.py", "criterion_4 or criterion_6 or criterion_7 or criterion_8"),
])
def test_reference_suite_passes_with_dropin(module, select, tmp_path):
    if not (REF_TESTS / module).exists():
        pytest.skip("reference not present (GPU box)")
    env = dict(os.environ, VATTN_REPO=str(ROOT), VATTN_REF=str(REF_SRC),
               PYTHONPATH=f"{ROOT / 'tests'}:{ROOT}:{REF_SRC}")
    cmd = [sys.executable, "-m", "pytest", str(REF_TESTS / module), "-q", "-p", "dropin_plugin",
           "-p", "no:cacheprovider", "-x"]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
