"""The C-ABI library loads on a CPU-only host and exports every symbol include/vattn.h declares
(no compute calls here), and the Python binding covers all of them."""

import ctypes as C
import re

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "vattn.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vattn_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2405_04437_b200._abi import LIB_PATH, lib

    lib()                                   # builds if needed, loads without a GPU
    raw = C.CDLL(str(LIB_PATH))
    names = _declared()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(raw, n)]
    assert missing == []


def test_python_binding_covers_header():
    from paper_2405_04437_b200._abi import SIGNATURES

    assert sorted(SIGNATURES) == _declared()


def test_shadow_backend_runs_without_gpu_and_cuda_backend_fails_loudly():
    import pytest
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.errors import CudaError

    g = ModelGeometry(2, 2, 64, 2, max_context=512, max_batch=2)
    m = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=16 << 20), backend="shadow")
    assert m.alloc_reqid() == 0
    assert m.step([100, 0]).ok
    m.close()
    if not torch.cuda.is_available():
        with pytest.raises((CudaError, RuntimeError)):
            KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=16 << 20), backend="cuda", device=0)


def test_abi_version():
    from paper_2405_04437_b200._abi import lib

    assert lib().vattn_abi_version() == 1
    assert lib().vattn_api_count() == 12


def test_struct_layouts_match_the_header():
    """The ctypes binding's structs have the C ABI's sizes (vattn_abi_sizes), so a field added
    to include/vattn.h without the binding (or vice versa) fails here, on CPU."""
    import ctypes as C

    from paper_2405_04437_b200 import _abi

    out = (C.c_int64 * 8)()
    assert _abi.lib().vattn_abi_sizes(out, 8) == 8
    mine = [C.sizeof(t) for t in (_abi.Config, _abi.Counters, _abi.StepResultC, _abi.BgResult,
                                   _abi.IterationResult, _abi.CacheDesc, _abi.RotaryC, _abi.LatencyEntry)]
    assert list(out) == mine


def test_phys_chunk_groups_plumbing_on_the_shadow_backend():
    """phys_chunk_groups reaches the core through the binding (counters echo it); the shadow
    backend has no physical memory, so its logical state is the reference's either way."""
    import pytest

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry

    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=2)
    states = []
    for chunk in (1, 4):
        m = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=64 << 20), backend="shadow",
                           phys_chunk_groups=chunk)
        c = m._counters()
        assert c.phys_chunk_groups == chunk and c.phys_mapped_bytes == 0
        r = m.alloc_reqid()
        assert m.step([3000 if i == r else 0 for i in range(2)]).ok
        states.append(m.parity_state())
        m.close()
    assert states[0] == states[1]
    with pytest.raises(ValueError):
        KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=64 << 20), backend="shadow",
                       phys_chunk_groups=0)
