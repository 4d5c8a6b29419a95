"""VATTN_CHECK_BOUNDS guard (attention.check_bounds): host-side check that every cache row a
kernel would touch is backed by a mapped page-group.  Runs on the shadow backend (no device)."""

import pytest

from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import check_bounds
from paper_2405_04437_b200.geometry import ModelGeometry

MB2 = 2 * 1024 * 1024


@pytest.fixture
def mgr():
    # 2 layers, 8 KV heads x 128: 2 KiB per token per buffer -> 1024 tokens per 2 MiB group
    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    m = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2), backend="shadow")
    yield m
    m.close()


def test_backed_rows_pass_and_unbacked_rows_raise(mgr):
    r0, r1 = mgr.alloc_reqid(), mgr.alloc_reqid()
    lens = [0] * 4
    lens[r0], lens[r1] = 1000, 1025          # 1 and 2 groups
    assert mgr.step(lens).ok
    check_bounds(mgr, [1000, 1025], [r0, r1])
    check_bounds(mgr, [1024, 2048], [r0, r1])            # the whole mapped prefix is usable
    check_bounds(mgr, [1023], [r0], extra_rows=1)        # fused append of one token
    with pytest.raises(ValueError, match="only 1024 are mapped"):
        check_bounds(mgr, [1024], [r0], extra_rows=1)
    with pytest.raises(ValueError, match="not a slot"):
        check_bounds(mgr, [1], [7])
    with pytest.raises(ValueError):
        check_bounds(mgr, [1], [2])                       # never stepped: nothing mapped
    with pytest.raises(ValueError):
        check_bounds(mgr, [-1], [r0])


def test_default_batch_index_is_identity(mgr):
    rids = [mgr.alloc_reqid() for _ in range(4)]
    assert rids == [0, 1, 2, 3]
    assert mgr.step([10, 20, 30, 40]).ok
    check_bounds(mgr, [10, 20, 30, 40])
    with pytest.raises(ValueError):
        check_bounds(mgr, [10, 20, 30, 1025])
