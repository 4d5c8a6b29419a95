"""GPU: the CTA-pair prefill kernel (tcgen05 cta_group::2, VATTN_PF_PAIR=1) against the
fp32 reference, in a subprocess because the kernel choice is read once per process."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_pair_kernel_matches_reference():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, VATTN_PF_PAIR="1")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "pf_pair_check.py"), "--parity-only"],
                       env=env, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if "max-normalised err" in ln]
    assert len(lines) == 5, r.stdout
    assert all(ln.endswith("OK") for ln in lines), r.stdout
