"""GPU: the persistent varlen prefill kernel (one CTA per SM walking the work list)
is bit-identical to the one-CTA-per-item kernel on short, long, mixed, prefixed and non-causal
prompt mixes, and within 2e-2 of the fp32 oracle on three requests of the mixed, prefixed and
non-causal ones.  Each kernel choice runs in its own process (VATTN_PF_PERSIST is read once)."""

import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_persistent_varlen_bit_equal_to_grid_kernel():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "pf_persist_varlen_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ALL BIT-EQUAL" in r.stdout, r.stdout[-3000:]
    assert r.stdout.count("bit-equal True") == 11, r.stdout[-3000:]
