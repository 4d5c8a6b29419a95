"""GPU cross-check against flash-attn 2.8.3, the kernel library vAttention targets
(SURVEY §8(c)).

* The paper's central claim: an UNMODIFIED non-paged kernel (`flash_attn_with_kvcache` with
  `cache_batch_idx`) runs directly on the virtual KV cache that the allocator backs on demand.
* Our decode, fused append+decode and prefill kernels follow the same conventions:
  * GQA mapping h -> h // (Hq/Hkv);
  * bottom-right causal alignment;
  * scale 1/sqrt(D);
  * k=/v= rows written at cache_seqlens[b].

Tolerance as in the rest of the suite: max|o - o_ref| / max|o_ref| <= 2e-2.  Both sides use
bf16 inputs and fp32 accumulation, so in practice the agreement is ~1e-3.  The appended cache
rows are compared bit-exactly.
"""

import pytest
import torch

from oracle.attention import max_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2
MB2 = 2 * 1024 * 1024


def _fa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return pytest.importorskip("flash_attn")


def _rand(shape, gen, dev):
    return torch.randn(shape, generator=gen).to(torch.bfloat16).to(dev)


def test_unmodified_flash_attn_runs_on_the_vmm_cache():
    fa = _fa()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention, kv_append
    from paper_2405_04437_b200.geometry import ModelGeometry

    dev = torch.device("cuda")
    g = ModelGeometry(n_layers=2, kv_heads_total=8, head_dim=128, bytes_per_elem=2, max_context=8192,
                      max_batch=8, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=1 << 30))
    try:
        gen = torch.Generator().manual_seed(11)
        rids = [mgr.alloc_reqid() for _ in range(5)]
        lens = [0] * g.max_batch
        for rid, n in zip(rids, (1, 1023, 1024, 1025, 5000)):
            lens[rid] = n
        assert mgr.step(lens).ok
        for layer in range(g.n_layers):
            for rid in rids:
                n = lens[rid]
                kv_append(mgr, layer, _rand((1, n, 8, 128), gen, dev), _rand((1, n, 8, 128), gen, dev),
                          torch.zeros(1, dtype=torch.int32, device=dev),
                          torch.tensor([rid], dtype=torch.int32, device=dev))
        # a permuted batch order exercises cache_batch_idx
        order = [rids[i] for i in (3, 0, 4, 2, 1)]
        idx = torch.tensor(order, dtype=torch.int32, device=dev)
        seq = torch.tensor([lens[r] for r in order], dtype=torch.int32, device=dev)
        q = _rand((5, 32, 128), gen, dev)
        for layer in range(g.n_layers):
            ours = decode_attention(mgr, layer, q, seq, idx)
            ref = fa.flash_attn_with_kvcache(q.unsqueeze(1), mgr.k_cache(layer), mgr.v_cache(layer),
                                             cache_seqlens=seq, cache_batch_idx=idx).squeeze(1)
            torch.cuda.synchronize()
            assert torch.isfinite(ref.float()).all()
            assert max_rel_err(ours.float().cpu(), ref.float().cpu()) <= TOL
    finally:
        mgr.close()


@pytest.mark.parametrize("splits", [0, 3])
def test_fused_append_decode_matches_flash_attn_kvcache(splits):
    fa = _fa()
    from paper_2405_04437_b200.attention import decode_attention_append_raw

    dev = torch.device("cuda")
    gen = torch.Generator().manual_seed(12)
    B, hq, hkv, d, L = 6, 56, 8, 128, 2048
    kc, vc = _rand((B + 2, L, hkv, d), gen, dev), _rand((B + 2, L, hkv, d), gen, dev)
    lens = torch.tensor([0, 1, 63, 64, 700, 2047], dtype=torch.int32, device=dev)   # before the token
    idx = torch.tensor([7, 0, 3, 1, 6, 2], dtype=torch.int32, device=dev)
    q = _rand((B, hq, d), gen, dev)
    kn, vn = _rand((B, hkv, d), gen, dev), _rand((B, hkv, d), gen, dev)
    k_fa, v_fa = kc.clone(), vc.clone()
    ref = fa.flash_attn_with_kvcache(q.unsqueeze(1), k_fa, v_fa, k=kn.unsqueeze(1), v=vn.unsqueeze(1),
                                     cache_seqlens=lens, cache_batch_idx=idx).squeeze(1)
    ours = decode_attention_append_raw(q, kc, vc, kn, vn, lens, idx, num_splits=splits)
    torch.cuda.synchronize()
    assert max_rel_err(ours.float().cpu(), ref.float().cpu()) <= TOL
    assert torch.equal(kc, k_fa) and torch.equal(vc, v_fa)


@pytest.mark.parametrize("n_q,kv_len,causal", [(1000, 1000, True), (300, 1100, True), (4096, 4096, True),
                                               (777, 777, False)])
def test_prefill_matches_flash_attn(n_q, kv_len, causal):
    fa = _fa()
    from paper_2405_04437_b200.attention import prefill_attention_raw

    dev = torch.device("cuda")
    gen = torch.Generator().manual_seed(13)
    hq, hkv, d, slot = 32, 4, 128, 1
    L = (kv_len + 127) // 128 * 128
    kc, vc = _rand((3, L, hkv, d), gen, dev), _rand((3, L, hkv, d), gen, dev)
    q = _rand((n_q, hq, d), gen, dev)
    ref = fa.flash_attn_func(q.unsqueeze(0), kc[slot:slot + 1, :kv_len], vc[slot:slot + 1, :kv_len],
                             causal=causal).squeeze(0)
    ours = prefill_attention_raw(q, kc, vc, slot, kv_len, causal=causal)
    torch.cuda.synchronize()
    assert max_rel_err(ours.float().cpu(), ref.float().cpu()) <= TOL


@pytest.mark.parametrize("interleaved", [False, True])
def test_rotary_fused_decode_matches_flash_attn_on_the_vmm_cache(interleaved):
    """Manager-backed fused append+decode with rotary vs flash_attn_with_kvcache(k=, v=,
    rotary_cos=, rotary_sin=, rotary_interleaved=) on two copies of the same VMM-backed cache."""
    fa = _fa()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append, kv_append
    from paper_2405_04437_b200.geometry import ModelGeometry

    dev = torch.device("cuda")
    g = ModelGeometry(n_layers=2, kv_heads_total=8, head_dim=128, bytes_per_elem=2, max_context=4096,
                      max_batch=4, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=1 << 30))
    try:
        gen = torch.Generator().manual_seed(12)
        rids = [mgr.alloc_reqid() for _ in range(3)]
        lens = [0] * 4
        for rid, n in zip(rids, (100, 1023, 2500)):
            lens[rid] = n + 1
        assert mgr.step(lens).ok
        for layer in range(2):      # layer 0 = ours, layer 1 = flash-attn; same history
            gl = torch.Generator().manual_seed(13)
            for rid in rids:
                n = lens[rid] - 1
                kv_append(mgr, layer, _rand((1, n, 8, 128), gl, dev), _rand((1, n, 8, 128), gl, dev),
                          torch.zeros(1, dtype=torch.int32, device=dev),
                          torch.tensor([rid], dtype=torch.int32, device=dev))
        idx = torch.tensor(rids, dtype=torch.int32, device=dev)
        seq = torch.tensor([lens[r] - 1 for r in rids], dtype=torch.int32, device=dev)
        q = _rand((3, 32, 128), gen, dev)
        kn, vn = _rand((3, 8, 128), gen, dev), _rand((3, 8, 128), gen, dev)
        ang = torch.arange(4096, dtype=torch.float32)[:, None] / (10000 ** (torch.arange(0, 128, 2) / 128))[None, :]
        cos, sin = ang.cos().to(dev), ang.sin().to(dev)
        ours = decode_attention_append(mgr, 0, q, kn, vn, seq, idx, rotary_cos=cos, rotary_sin=sin,
                                       rotary_interleaved=interleaved)
        ref = fa.flash_attn_with_kvcache(q.unsqueeze(1), mgr.k_cache(1), mgr.v_cache(1), k=kn.unsqueeze(1),
                                         v=vn.unsqueeze(1), rotary_cos=cos.to(torch.bfloat16),
                                         rotary_sin=sin.to(torch.bfloat16), cache_seqlens=seq,
                                         cache_batch_idx=idx, rotary_interleaved=interleaved).squeeze(1)
        torch.cuda.synchronize()
        assert max_rel_err(ours.float().cpu(), ref.float().cpu()) <= TOL
        for i, r in enumerate(rids):   # both caches hold the rotated new k (bf16 tables on the flash-attn side)
            p = lens[r] - 1
            assert torch.allclose(mgr.k_cache(0)[r, p].float(), mgr.k_cache(1)[r, p].float(), rtol=2e-2, atol=2e-2)
    finally:
        mgr.close()
