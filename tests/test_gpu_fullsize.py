"""Parity at BASELINE full sizes through size-independent properties (the fp32 oracle is too
slow there): the virtual-memory cache behaves exactly like plain device memory, the paged
layout computes bit-identical attention, and split-K is consistent."""

import pytest
import torch

from oracle.attention import decode_ref, max_rel_err

pytestmark = pytest.mark.gpu
MB2 = 2 * 1024 * 1024


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


def test_l8_full_layer_vmm_cache_equals_plain_memory():
    """BASELINE config 2 layer (B 64, ctx 4096, 32 Q / 8 KV heads): fused append+decode on the
    cuMem-backed virtual cache == the same kernel on a cudaMalloc copy, bit for bit; sampled
    rows checked against the fp32 oracle."""
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append, decode_attention_append_raw, kv_append
    from paper_2405_04437_b200.geometry import llama3_8b

    dev = _cuda()
    g = llama3_8b(max_context=8192, max_batch=64)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * 2 * 5 * MB2))
    rids = [mgr.alloc_reqid() for _ in range(64)]
    ctx = 4096
    assert mgr.step([ctx + 1] * 64).ok
    gen = torch.Generator(device=dev).manual_seed(0)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    for c0 in range(0, ctx, 1024):
        kn = torch.randn(64, 1024, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        vn = torch.randn_like(kn)
        kv_append(mgr, 0, kn, vn, torch.full((64,), c0, dtype=torch.int32, device=dev), idx)
    backed = mgr.slots[rids[0]].mapped_groups * (MB2 // g.per_token_layer_bytes)   # rows behind pages
    k_plain = torch.zeros(64, 8192, 8, 128, device=dev, dtype=torch.bfloat16)
    v_plain = torch.zeros_like(k_plain)
    k_plain[:, :backed] = mgr.k_cache(0)[:, :backed]     # only backed rows may be touched
    v_plain[:, :backed] = mgr.v_cache(0)[:, :backed]
    q = torch.randn(64, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    k1 = torch.randn(64, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    v1 = torch.randn_like(k1)
    pos = torch.full((64,), ctx, dtype=torch.int32, device=dev)
    out_vmm = decode_attention_append(mgr, 0, q, k1, v1, pos, idx)
    out_plain = decode_attention_append_raw(q, k_plain, v_plain, k1, v1, pos, idx)
    torch.cuda.synchronize()
    assert torch.equal(out_vmm, out_plain)
    assert torch.equal(mgr.k_cache(0)[:, : ctx + 1], k_plain[:, : ctx + 1])
    for b in (0, 37, 63):                       # sampled rows vs the fp32 oracle
        r = rids[b]
        ref = decode_ref(q[b:b + 1].cpu(), k_plain[r:r + 1, : ctx + 1].cpu(), v_plain[r:r + 1, : ctx + 1].cpu(),
                         torch.tensor([ctx + 1], dtype=torch.int32))
        assert max_rel_err(out_vmm[b:b + 1].cpu(), ref) <= 2e-2
    mgr.close()


def test_l8_full_layer_paged_equals_contiguous_and_splits_agree():
    from paper_2405_04437_b200.attention import decode_attention_paged, decode_attention_raw

    dev = _cuda()
    B, hq, hkv, L = 64, 32, 8, 4096
    gen = torch.Generator(device=dev).manual_seed(1)
    k = torch.randn(B, L, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    q = torch.randn(B, hq, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    seq = torch.randint(1, L + 1, (B,), device=dev, generator=gen, dtype=torch.int32)
    base = decode_attention_raw(q, k, v, seq, num_splits=1)
    for bs in (16, 256):
        nb = L // bs
        perm = torch.randperm(B * nb, device=dev, generator=gen)
        kp = torch.empty_like(k).view(B * nb, bs, hkv, 128)
        vp = torch.empty_like(v).view(B * nb, bs, hkv, 128)
        kp[perm] = k.view(B * nb, bs, hkv, 128)
        vp[perm] = v.view(B * nb, bs, hkv, 128)
        out = decode_attention_paged(q, kp, vp, perm.view(B, nb).to(torch.int32), seq, num_splits=1)
        assert torch.equal(out, base)
    for s in (2, 5):                              # split-K + LSE combine stays within tolerance
        out = decode_attention_raw(q, k, v, seq, num_splits=s)
        assert max_rel_err(out.float().cpu(), base.float().cpu()) <= 1e-2


def test_pdl_layer_chain_equals_serial_launches():
    """Decode launches are programmatic dependents of the previous kernel on the stream: a layer's
    K/V stream starts under the previous layer's tail (kv_early), but never when the previous
    launch appended to the SAME layer.  Back-to-back fused launches over 4 layers, then a plain
    decode of the last layer that must see the row its predecessor appended, all bit-equal to the
    raw-path kernels (which always wait) on plain-memory copies."""
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import (decode_attention, decode_attention_append, decode_attention_append_raw,
                                                 decode_attention_raw, kv_append)
    from paper_2405_04437_b200.geometry import ModelGeometry

    dev = _cuda()
    N, B, ctx = 4, 16, 2000
    g = ModelGeometry(N, 8, 128, 2, max_context=4096, max_batch=B, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=2 * N * B * 2 * MB2))
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([ctx + 2] * B).ok
    gen = torch.Generator(device=dev).manual_seed(17)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    zero = torch.zeros(B, dtype=torch.int32, device=dev)
    for layer in range(N):
        kv = torch.randn(B, ctx, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kv_append(mgr, layer, kv, kv * 0.5, zero, idx)
    q = torch.randn(N, B, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    k1 = torch.randn(N, B, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    plain = [(mgr.k_cache(l)[rids, :ctx + 2].clone(), mgr.v_cache(l)[rids, :ctx + 2].clone()) for l in range(N)]
    outs = [decode_attention_append(mgr, l, q[l], k1[l], k1[l] * 2, pos, idx, num_splits=s)
            for l, s in zip(range(N), (1, 3, 0, 2))]
    again = decode_attention(mgr, N - 1, q[0], pos + 1, idx)          # same layer as its predecessor
    torch.cuda.synchronize()
    for l, s in zip(range(N), (1, 3, 0, 2)):
        kp, vp = plain[l]
        want = decode_attention_append_raw(q[l], kp, vp, k1[l], k1[l] * 2, pos, num_splits=s)
        torch.cuda.synchronize()
        assert torch.equal(outs[l], want), l
    kp, vp = plain[N - 1]
    assert torch.equal(again, decode_attention_raw(q[0], kp, vp, pos + 1))
    mgr.close()
