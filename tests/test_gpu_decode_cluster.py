"""GPU: decode split-K merged inside the cluster of a unit's splits over DSMEM (default for 2-8
splits) is bit-identical to the separate combine kernel (VATTN_DEC_CLUSTER=0) and within the
north-star tolerance of the fp32 oracle (tools/dec_cluster_check.py: empty rows, D 64/128, GQA
4-8, plain and fused-append decode).  Subprocesses, since the mode is read once per process."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _run(cluster: str) -> list[str]:
    env = dict(os.environ, VATTN_DEC_CLUSTER=cluster)
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "dec_cluster_check.py")], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.startswith("case ")]


def test_cluster_combine_bit_identical_to_combine_kernel():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    a, b = _run("1"), _run("0")
    assert len(a) == 8 and a == b, (a, b)
    for ln in a:
        assert float(ln.rsplit("err ", 1)[1]) <= 2e-2, ln
