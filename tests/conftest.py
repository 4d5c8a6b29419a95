import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))

REF_SRC = Path(os.environ.get("VATTN_REF", "/root/reference/pkg/src"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ref_kvsim():
    """The reference package itself, importable only in the build container."""
    if not (REF_SRC / "kvsim").is_dir():
        pytest.skip("reference not present (GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import kvsim
    return kvsim
