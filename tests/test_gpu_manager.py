"""GPU: the allocator with the real CUDA VMM backend (cuMemAddressReserve / cuMemCreate /
cuMemMap / cuMemSetAccess at 2 MiB) — bookkeeping parity against the reference recordings,
and the kernels running on the resulting virtual tensors."""

import pytest
import torch

from allocator_replay import CoreAdapter, load_fixtures, replay
from oracle.attention import decode_ref, max_rel_err

pytestmark = pytest.mark.gpu

MB2 = 2 * 1024 * 1024
GPU_FIXTURES = [f for f in load_fixtures()
                if f["config"]["page_group_size"] == MB2 and f["config"]["pool_bytes"] <= 8 * 1024 ** 3]


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("fixture", GPU_FIXTURES, ids=[f["name"] for f in GPU_FIXTURES])
def test_cuda_backend_bookkeeping_matches_reference(fixture):
    _cuda()
    a = CoreAdapter(fixture, backend="cuda")
    try:
        replay(fixture, a)
        st = a.m.driver_stats()
        # every shadow map was a real cuMemMap (+ coalesced cuMemSetAccess)
        assert st["real_maps"] == a.m.vmm.calls.get("cuMemMap", 0)
        assert st["real_unmaps"] == a.m.vmm.calls.get("cuMemUnmap", 0)
    finally:
        a.close()


@pytest.mark.parametrize("release", [False, True], ids=["recycle", "release"])
@pytest.mark.parametrize("fixture", GPU_FIXTURES[::3], ids=[f["name"] for f in GPU_FIXTURES[::3]])
def test_cuda_backend_chunked_bookkeeping_matches_reference(fixture, release):
    """phys_chunk_groups=4: four consecutive 2 MiB groups of a buffer share one 8 MiB physical
    handle.  The logical state after every reference call is unchanged (bit-exact replay); the
    driver sees at most as many cuMemMap calls as the 2 MiB mode, and the mapped chunks cover
    every logically mapped group."""
    _cuda()
    a = CoreAdapter(fixture, backend="cuda", phys_chunk_groups=4, release_physical=release)
    try:
        replay(fixture, a)
        st = a.m.driver_stats()
        c = a.m._counters()
        assert c.phys_chunk_groups == 4
        assert st["real_maps"] <= a.m.vmm.calls.get("cuMemMap", 0)
        assert c.phys_mapped_bytes >= c.mapped * c.page_group_size
        assert c.phys_chunks_mapped * 4 * MB2 >= c.phys_mapped_bytes
    finally:
        a.close()


def test_chunked_cache_data_survives_neighbour_unmaps():
    """Chunk mode on a real cache: rows written while their group shares a chunk with groups that
    are later trimmed/reclaimed keep their values; decode over them equals the 2 MiB-mode result
    bit for bit, with fewer driver maps."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention, kv_append

    dev = torch.device("cuda")
    g = ModelGeometry(2, 8, 128, 2, max_context=16384, max_batch=4, n_q_heads_total=32)
    outs, maps = [], []
    for chunk in (1, 4):
        mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=256 * MB2, reclaim_threshold=0.0),
                             phys_chunk_groups=chunk)
        gen = torch.Generator(device=dev).manual_seed(5)
        rids = [mgr.alloc_reqid() for _ in range(3)]
        lens = [0] * 4
        for r, n in zip(rids, (5000, 3000, 9000)):
            lens[r] = n
        assert mgr.step(lens).ok
        idx = torch.tensor(rids, dtype=torch.int32, device=dev)
        for layer in range(2):
            for r in rids:
                n = lens[r]
                kv = torch.randn(1, n, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
                kv_append(mgr, layer, kv, kv, torch.zeros(1, dtype=torch.int32, device=dev),
                          torch.tensor([r], dtype=torch.int32, device=dev))
        # free the middle request and shrink the first: their groups (and maybe chunks) go
        mgr.free_reqid(rids[1])
        lens[rids[1]] = 0
        lens[rids[0]] = 2100
        assert mgr.step(lens).ok
        mgr.reclaim()
        q = torch.randn(2, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        sel = torch.tensor([rids[0], rids[2]], dtype=torch.int32, device=dev)
        seq = torch.tensor([lens[rids[0]], lens[rids[2]]], dtype=torch.int32, device=dev)
        o = [decode_attention(mgr, layer, q, seq, sel) for layer in range(2)]
        torch.cuda.synchronize()
        mgr.check_errors()
        outs.append(torch.stack(o).cpu())
        maps.append(mgr.driver_stats()["real_maps"])
        mgr.close()
    assert torch.equal(outs[0], outs[1])
    assert maps[1] < maps[0]


def test_tiny_config_end_to_end():
    """BASELINE config 1: 1 layer, 8 Q / 2 KV heads, D 64, batch 2, contexts 128-512, 2 MiB."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention, kv_append
    from paper_2405_04437_b200.geometry import tiny

    dev = torch.device("cuda")
    g = tiny()
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * 1024 * 1024))
    r0, r1 = mgr.alloc_reqid(), mgr.alloc_reqid()
    lens = [0, 0]
    lens[r0], lens[r1] = 128, 512
    assert mgr.step(lens).ok
    assert mgr.vmm.pool.mapped == 2 * 2      # 1 group per slot x 2 buffers
    gen = torch.Generator().manual_seed(0)
    for rid in (r0, r1):
        n = lens[rid]
        kn = torch.randn(1, n, 2, 64, generator=gen).to(torch.bfloat16)
        vn = torch.randn(1, n, 2, 64, generator=gen).to(torch.bfloat16)
        kv_append(mgr, 0, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
                  torch.tensor([rid], dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    kc, vc = mgr.k_cache(0), mgr.v_cache(0)
    q = torch.randn(2, 8, 64, generator=gen).to(torch.bfloat16)
    seq = torch.tensor([lens[r0], lens[r1]], dtype=torch.int32)
    idx = torch.tensor([r0, r1], dtype=torch.int32)
    k_host = torch.zeros(2, 512, 2, 64, dtype=torch.bfloat16)
    v_host = torch.zeros_like(k_host)
    for rid in (r0, r1):
        k_host[rid, : lens[rid]] = kc[rid, : lens[rid]].cpu()
        v_host[rid, : lens[rid]] = vc[rid, : lens[rid]].cpu()
    ref = decode_ref(q, k_host, v_host, seq, idx)
    out = decode_attention(mgr, 0, q.to(dev), seq.to(dev), idx.to(dev))
    torch.cuda.synchronize()
    assert max_rel_err(out.cpu(), ref) <= 2e-2
    mgr.close()


def test_decode_through_manager_l8_shape_with_growth():
    """L8 geometry (reduced batch/layers): decode steps cross a 1024-token page boundary; the
    background thread maps the next page during the previous step's kernels."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention, kv_append

    dev = torch.device("cuda")
    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=256 * MB2))
    rids = [mgr.alloc_reqid() for _ in range(3)]
    lens = [0] * 4
    for i, r in enumerate(rids):
        lens[r] = 1020 + i
    assert mgr.step(lens).ok
    gen = torch.Generator().manual_seed(5)
    host_k = {l: torch.zeros(4, 4096, 8, 128, dtype=torch.bfloat16) for l in range(2)}
    host_v = {l: torch.zeros(4, 4096, 8, 128, dtype=torch.bfloat16) for l in range(2)}
    for layer in range(2):
        for r in rids:
            kn = torch.randn(1, lens[r], 8, 128, generator=gen).to(torch.bfloat16)
            vn = torch.randn(1, lens[r], 8, 128, generator=gen).to(torch.bfloat16)
            host_k[layer][r, : lens[r]] = kn[0]
            host_v[layer][r, : lens[r]] = vn[0]
            kv_append(mgr, layer, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
                      torch.tensor([r], dtype=torch.int32, device=dev))
    idx = torch.tensor(rids, dtype=torch.int32)
    for it in range(8):
        nxt = list(lens)
        for r in rids:
            nxt[r] += 1
        plan = mgr.plan_overlap(nxt)
        mgr.bg_submit(plan)                    # maps crossing pages while we append+decode
        res = mgr.step(nxt)                    # joins the window; nothing left to map
        assert res.ok and res.sync_us == 0.0
        seq_before = torch.tensor([lens[r] for r in rids], dtype=torch.int32)
        seq_after = seq_before + 1
        for layer in range(2):
            kn = torch.randn(3, 8, 128, generator=gen).to(torch.bfloat16)
            vn = torch.randn(3, 8, 128, generator=gen).to(torch.bfloat16)
            for j, r in enumerate(rids):
                host_k[layer][r, lens[r]] = kn[j]
                host_v[layer][r, lens[r]] = vn[j]
            kv_append(mgr, layer, kn.to(dev), vn.to(dev), seq_before.to(dev), idx.to(dev))
            q = torch.randn(3, 32, 128, generator=gen).to(torch.bfloat16)
            out = decode_attention(mgr, layer, q.to(dev), seq_after.to(dev), idx.to(dev))
            ref = decode_ref(q, host_k[layer], host_v[layer], seq_after, idx)
            torch.cuda.synchronize()
            assert max_rel_err(out.cpu(), ref) <= 2e-2, (it, layer)
        lens = nxt
    assert mgr.slots[rids[-1]].mapped_groups == 2     # 1022+8 tokens crossed 1024
    mgr.close()


@pytest.mark.parametrize("spec_slots,lazy,chunk", [(0, False, 1), (2, False, 1), (0, True, 1), (2, True, 1),
                                                   (2, True, 4), (0, False, 4)])
def test_physical_prefetch_keeps_logical_state_and_data(spec_slots, lazy, chunk):
    """Prefetch (and speculative eager) maps pages ahead of the reference schedule; the logical
    state must equal the oracle's after every call and kernels must read/write the adopted pages
    correctly."""
    _cuda()
    import random

    from oracle.allocator import Geometry, OracleManager
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention, kv_append

    dev = torch.device("cuda")
    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    pool = 24 * 4 * MB2
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=pool), prefetch_tokens=1500,
                         prefetch_slots=spec_slots, prefetch_slot_tokens=1800, lazy_unmap=lazy,
                         phys_chunk_groups=chunk)
    om = OracleManager(Geometry(2, 8, 128, 2, 4096, 4), MB2, pool_bytes=pool)
    rng = random.Random(0)
    gen = torch.Generator().manual_seed(9)
    host_k = torch.zeros(4, 4096, 8, 128, dtype=torch.bfloat16)
    host_v = torch.zeros_like(host_k)
    lens = [0] * 4
    for it in range(60):
        if it % 9 == 0 and 0 in lens:
            r = mgr.alloc_reqid()
            assert r == om.alloc_reqid()
            lens[r] = rng.randint(1, 900)
            new = {r: lens[r]}
        else:
            new = {}
            for r in range(4):
                if lens[r]:
                    add = rng.choice([1, 1, 64, 300])
                    if lens[r] + add <= 4096:
                        new[r] = add
                        lens[r] += add
        res = mgr.step(lens)
        ok, us = om.step(lens)
        assert (res.ok, res.sync_us) == (ok, us)
        for r, n in new.items():          # append the new rows of this step (layer 0)
            p0 = lens[r] - n
            kn = torch.randn(1, n, 8, 128, generator=gen).to(torch.bfloat16)
            vn = torch.randn(1, n, 8, 128, generator=gen).to(torch.bfloat16)
            host_k[r, p0:lens[r]] = kn[0]
            host_v[r, p0:lens[r]] = vn[0]
            kv_append(mgr, 0, kn.to(dev), vn.to(dev), torch.tensor([p0], dtype=torch.int32, device=dev),
                      torch.tensor([r], dtype=torch.int32, device=dev))
        act = [r for r in range(4) if lens[r]]
        q = torch.randn(len(act), 32, 128, generator=gen).to(torch.bfloat16)
        seq = torch.tensor([lens[r] for r in act], dtype=torch.int32)
        idx = torch.tensor(act, dtype=torch.int32)
        out = decode_attention(mgr, 0, q.to(dev), seq.to(dev), idx.to(dev))
        mgr.bg_submit(execute_plan=False, prefetch=True)   # speculative maps during the kernel
        ref = decode_ref(q, host_k, host_v, seq, idx)
        torch.cuda.synchronize()
        assert max_rel_err(out.cpu(), ref) <= 2e-2, it
        mgr.bg_wait()
        st = mgr.parity_state()
        assert st["mapped"] == om.dev.mapped and st["created"] == om.dev.created
        assert [s[2] for s in st["slots"]] == [s[2] for s in om.slots]
        if it % 13 == 12:                 # retire one
            r = max(act)
            mgr.free_reqid(r)
            om.free_reqid(r)
            lens[r] = 0
    ds = mgr.driver_stats()
    assert ds["spec_maps"] > 0 and ds["spec_hits"] > 0
    if lazy:
        assert ds["lazy_unmaps"] > 0 and ds["real_unmaps"] < ds["lazy_unmaps"]
    mgr.close()


def test_prefetch_hint_backs_the_predicted_slot_before_admission():
    """Staged admission: hint a queued prompt at the slot alloc_reqid will return; once the
    prefetch worker reports it ready, admitting it and stepping to the prompt length maps every
    page-group without a single driver call (all adopted), and the data path works."""
    _cuda()
    import time

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention, kv_append

    dev = torch.device("cuda")
    g = ModelGeometry(4, 8, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=96 * MB2, eager_groups=0),
                         lazy_unmap=True)
    r0 = mgr.alloc_reqid()
    assert mgr.step([1500 if i == r0 else 0 for i in range(4)]).ok
    pred = mgr.predict_alloc(2)
    assert len(pred) == 2 and r0 not in pred
    mgr.prefetch_hint(pred[:1], [3000])
    assert not mgr.slot_ready(pred[0], 3000)
    mgr.bg_submit(execute_plan=False, prefetch=True)
    t0 = time.time()
    while not mgr.slot_ready(pred[0], 3000):
        assert time.time() - t0 < 60, "prefetch worker did not back the hinted slot"
        time.sleep(0.01)
    before = mgr.driver_stats()
    r1 = mgr.alloc_reqid()
    assert r1 == pred[0]
    lens = [0] * 4
    lens[r0], lens[r1] = 1500, 3000
    assert mgr.step(lens).ok
    after = mgr.driver_stats()
    assert after["real_maps"] == before["real_maps"]          # every page adopted
    assert after["spec_hits"] - before["spec_hits"] == 3 * 8   # 3 groups x 8 buffers
    gen = torch.Generator().manual_seed(4)
    kn = torch.randn(1, 3000, 8, 128, generator=gen).to(torch.bfloat16)
    kv_append(mgr, 3, kn.to(dev), kn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
              torch.tensor([r1], dtype=torch.int32, device=dev))
    q = torch.randn(1, 32, 128, generator=gen).to(torch.bfloat16)
    out = decode_attention(mgr, 3, q.to(dev), torch.tensor([3000], dtype=torch.int32, device=dev),
                           torch.tensor([r1], dtype=torch.int32, device=dev))
    host = torch.zeros(4, 4096, 8, 128, dtype=torch.bfloat16)
    host[r1, :3000] = kn[0]
    ref = decode_ref(q, host, host, torch.tensor([3000], dtype=torch.int32), torch.tensor([r1], dtype=torch.int32))
    torch.cuda.synchronize()
    assert max_rel_err(out.cpu(), ref) <= 2e-2
    mgr.close()


def test_sliced_layout_kernels():
    """Layer-sliced layout ([B, L, N, H, D], manager.py:93-96): two buffers,
    token stride N·H·D·P; the same kernels serve it through the layer view."""
    _cuda()
    from oracle.attention import prefill_ref
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention_append, kv_append, prefill_attention

    dev = torch.device("cuda")
    g = ModelGeometry(4, 4, 128, 2, max_context=2048, max_batch=3, n_q_heads_total=16)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2, sliced=True))
    assert mgr.buffer_count == 2
    r = mgr.alloc_reqid()
    lens = [0, 0, 0]
    S = 700
    lens[r] = S + 1
    assert mgr.step(lens).ok
    gen = torch.Generator().manual_seed(4)
    for layer in range(4):
        kn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
        vn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
        q = torch.randn(S, 16, 128, generator=gen).to(torch.bfloat16)
        kv_append(mgr, layer, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
                  torch.tensor([r], dtype=torch.int32, device=dev))
        out = prefill_attention(mgr, layer, q.to(dev), r)
        torch.cuda.synchronize()
        assert max_rel_err(out.cpu(), prefill_ref(q, kn[0], vn[0])) <= 2e-2
        # decode one more token with the fused kernel
        k1 = torch.randn(1, 4, 128, generator=gen).to(torch.bfloat16)
        v1 = torch.randn(1, 4, 128, generator=gen).to(torch.bfloat16)
        q1 = torch.randn(1, 16, 128, generator=gen).to(torch.bfloat16)
        o1 = decode_attention_append(mgr, layer, q1.to(dev), k1.to(dev), v1.to(dev),
                                     torch.tensor([S], dtype=torch.int32, device=dev),
                                     torch.tensor([r], dtype=torch.int32, device=dev))
        kc = torch.cat([kn[0], k1], 0).unsqueeze(0)
        vc = torch.cat([vn[0], v1], 0).unsqueeze(0)
        ref = decode_ref(q1, kc, vc, torch.tensor([S + 1], dtype=torch.int32))
        torch.cuda.synchronize()
        assert max_rel_err(o1.cpu(), ref) <= 2e-2
        # the view sees the sliced strides
        assert torch.equal(mgr.k_cache(layer)[r, :S].cpu(), kn[0])
    mgr.close()
    # 3 layers: a 3 KiB token row does not tile a 2 MiB page-group into 64-token boxes (682.67
    # tokens per group), so a decode box could reach an unmapped page: the kernels load each row's
    # partial last tile with bounded per-row loads (CacheView::tail_guard) and match the oracle
    from paper_2405_04437_b200.attention import decode_attention
    g3 = ModelGeometry(3, 4, 128, 2, max_context=2048, max_batch=3, n_q_heads_total=16)
    m3 = KVCacheManager(g3, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2, sliced=True))
    r3 = m3.alloc_reqid()
    n3 = 682                                    # the last whole token of page-group 0
    assert m3.step([n3 if i == r3 else 0 for i in range(3)]).ok
    assert m3.slots[r3].mapped_groups == 1
    k3 = torch.randn(1, n3, 4, 128, generator=gen).to(torch.bfloat16)
    kv_append(m3, 2, k3.to(dev), k3.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
              torch.tensor([r3], dtype=torch.int32, device=dev))
    q3 = torch.randn(1, 16, 128, generator=gen).to(torch.bfloat16)
    o3 = decode_attention(m3, 2, q3.to(dev), torch.tensor([n3], dtype=torch.int32, device=dev),
                          torch.tensor([r3], dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    assert max_rel_err(o3.cpu(), decode_ref(q3, k3, k3, torch.tensor([n3], dtype=torch.int32))) <= 2e-2
    m3.close()


def test_bounds_guard_raises_instead_of_faulting(monkeypatch):
    """VATTN_CHECK_BOUNDS: a length past the mapped prefix is a ValueError, not a GPU fault."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, attention
    from paper_2405_04437_b200.geometry import ModelGeometry

    monkeypatch.setattr(attention, "CHECK_BOUNDS", True)
    dev = torch.device("cuda")
    g = ModelGeometry(1, 8, 128, 2, max_context=8192, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=16 * MB2))
    try:
        r = mgr.alloc_reqid()
        lens = [0, 0]
        lens[r] = 1000
        assert mgr.step(lens).ok                     # one 2 MiB group = 1024 tokens mapped
        q = torch.randn(1, 32, 128, device=dev, dtype=torch.bfloat16)
        idx = torch.tensor([r], dtype=torch.int32, device=dev)
        kv = torch.randn(1, 1024, 8, 128, device=dev, dtype=torch.bfloat16)   # fresh pages hold garbage
        attention.kv_append(mgr, 0, kv, kv, torch.zeros(1, dtype=torch.int32, device=dev), idx)
        with pytest.raises(ValueError, match="mapped"):
            attention.decode_attention(mgr, 0, q, torch.tensor([5000], dtype=torch.int32, device=dev), idx)
        out = attention.decode_attention(mgr, 0, q, torch.tensor([1024], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
    finally:
        mgr.close()


def test_foreground_window_holds_the_prefetch_worker():
    """vattn_set_foreground: while the caller is in its launch window the worker makes no new
    driver call; hinted pages appear only after the window closes."""
    _cuda()
    import time

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry

    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2, eager_groups=0),
                         lazy_unmap=True)
    (slot,) = mgr.predict_alloc(1)
    mgr.foreground(True)
    mgr.prefetch_hint([slot], [3000])
    mgr.bg_submit(execute_plan=False, prefetch=True)
    time.sleep(0.3)
    assert not mgr.slot_ready(slot, 3000)
    assert mgr.driver_stats()["spec_maps"] == 0
    mgr.foreground(False)
    t0 = time.time()
    while not mgr.slot_ready(slot, 3000):
        assert time.time() - t0 < 60
        time.sleep(0.01)
    assert mgr.driver_stats()["spec_maps"] == 3 * 4     # 3 groups x 4 buffers
    mgr.close()


def test_device_read_guard_clamps_and_raises_without_faulting():
    """Default-on device guard: lengths past a slot's backed rows, a slot
    index out of range, and appends past the backed rows are clamped / skipped by the kernels,
    which report through host-mapped words; the next call on the manager raises ValueError and
    the CUDA context stays usable.  Prefill (host kv_len) is refused before launch."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, attention
    from paper_2405_04437_b200.geometry import ModelGeometry

    dev = torch.device("cuda")
    g = ModelGeometry(1, 8, 128, 2, max_context=8192, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=16 * MB2))
    try:
        r = mgr.alloc_reqid()
        lens = [0, 0]
        lens[r] = 1000
        assert mgr.step(lens).ok                     # one 2 MiB group = 1024 rows backed
        gen = torch.Generator(device=dev).manual_seed(9)
        q = torch.randn(1, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        idx = torch.tensor([r], dtype=torch.int32, device=dev)
        kv = torch.randn(1, 1024, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        attention.kv_append(mgr, 0, kv, kv, torch.zeros(1, dtype=torch.int32, device=dev), idx)
        good = attention.decode_attention(mgr, 0, q, torch.tensor([1024], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        mgr.check_errors()
        # 1) a length past the backed rows: clamped to 1024 (same result), reported
        bad = attention.decode_attention(mgr, 0, q, torch.tensor([7000], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        assert torch.equal(bad, good)
        with pytest.raises(ValueError, match="backed rows"):
            mgr.check_errors()
        mgr.check_errors()                           # reported once
        # 2) a slot index out of range: no reads, zeros, reported at the next allocator call
        z = attention.decode_attention(mgr, 0, q, torch.tensor([10], dtype=torch.int32, device=dev),
                                       torch.tensor([5], dtype=torch.int32, device=dev))
        torch.cuda.synchronize()
        assert z.abs().max().item() == 0
        with pytest.raises(ValueError, match="backed rows"):
            mgr.step(lens)
        assert mgr.step(lens).ok
        # 3) fused append at a row that is not backed: the row is not written, reported
        k1 = torch.randn(1, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        attention.decode_attention_append(mgr, 0, q, k1, k1, torch.tensor([1024], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        with pytest.raises(ValueError):
            mgr.check_errors()
        # 4) plain append past the backed rows: skipped, reported
        attention.kv_append(mgr, 0, kv[:, :8], kv[:, :8], torch.tensor([1020], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        with pytest.raises(ValueError):
            mgr.check_errors()
        # rows 1020..1023 are backed and were written; 1024..1027 were skipped
        assert torch.equal(mgr.k_cache(0)[r, 1020:1024].cpu(), kv[0, :4].cpu())
        # 5) prefill with kv_len past the backed rows is refused on the host
        with pytest.raises(ValueError, match="backs"):
            attention.prefill_attention(mgr, 0, torch.zeros(2000, 32, 128, device=dev, dtype=torch.bfloat16), r)
        # the context is healthy: restore rows 1020..1023 (step 4 overwrote them) and a normal
        # decode matches the first one bit for bit
        attention.kv_append(mgr, 0, kv[:, 1020:], kv[:, 1020:], torch.tensor([1020], dtype=torch.int32, device=dev), idx)
        again = attention.decode_attention(mgr, 0, q, torch.tensor([1024], dtype=torch.int32, device=dev), idx)
        torch.cuda.synchronize()
        assert torch.equal(again, good)
        mgr.check_errors()
    finally:
        mgr.close()
