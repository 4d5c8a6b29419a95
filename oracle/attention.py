"""ORACLE — test infrastructure only, never the product path.

fp32 CPU restatement of the attention / KV-append semantics the build implements.  The
reference package has NO attention code, so these follow the paper:

* eq. 2  Attention(q, K, V) = softmax(q Kᵀ · scale) V
* K/V cache per layer laid out token-major [B, L, H, D]
* `cache_batch_idx` maps batch row b to cache slot
* Q/KV head counts (GQA), Table 5

and the third-party conventions the paper relies on without vendoring them (FlashAttention-2
v2.5.9 `flash_attn_with_kvcache`): query head h reads KV head h // (Hq/Hkv);
causal masking is bottom-right aligned (query i of an Sq-row block over Sk keys sees keys
j <= i + Sk - Sq); default scale 1/sqrt(D); `cache_seqlens` is the cache length before the
append of new rows.  Parity for attention is therefore "unpinned by the reference": the
tolerance is the north_star's (bf16 in, fp32 accumulate, max-rel-err <= 2e-2).

All functions take torch CPU tensors (any float dtype) and compute in float32.
"""

from __future__ import annotations

import math

import torch


def kv_append_ref(k_cache, v_cache, k_new, v_new, cache_seqlens, cache_batch_idx=None):
    """Write rows i of k_new[b] at position cache_seqlens[b] + i of slot cache_batch_idx[b].

    k_cache: [B_cache, L, Hkv, D]; k_new: [B, T, Hkv, D].  Returns updated copies.
    """
    k_out, v_out = k_cache.clone(), v_cache.clone()
    batch, n_new = k_new.shape[0], k_new.shape[1]
    for b in range(batch):
        slot = int(cache_batch_idx[b]) if cache_batch_idx is not None else b
        p0 = int(cache_seqlens[b])
        k_out[slot, p0:p0 + n_new] = k_new[b].to(k_out.dtype)
        v_out[slot, p0:p0 + n_new] = v_new[b].to(v_out.dtype)
    return k_out, v_out


def decode_ref(q, k_cache, v_cache, cache_seqlens, cache_batch_idx=None, scale=None):
    """One query token per batch row over the first cache_seqlens[b] cached tokens.

    q: [B, Hq, D]; k_cache/v_cache: [B_cache, L, Hkv, D].  Returns fp32 [B, Hq, D].
    Rows with cache_seqlens == 0 produce zeros (empty softmax).
    """
    batch, hq, d = q.shape
    hkv = k_cache.shape[2]
    group = hq // hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = torch.zeros(batch, hq, d, dtype=torch.float32)
    for b in range(batch):
        slot = int(cache_batch_idx[b]) if cache_batch_idx is not None else b
        n = int(cache_seqlens[b])
        if n == 0:
            continue
        k = k_cache[slot, :n].float()                  # [n, Hkv, D]
        v = v_cache[slot, :n].float()
        qb = q[b].float().view(hkv, group, d)          # head h -> kv head h // group
        s = torch.einsum("hgd,nhd->hgn", qb, k) * scale
        p = torch.softmax(s, dim=-1)
        out[b] = torch.einsum("hgn,nhd->hgd", p, v).reshape(hq, d)
    return out


def decode_ref_equal(q, k_cache, v_cache, n: int, scale=None, rows_per_chunk: int = 1):
    """decode_ref for a batch whose rows all attend over their first n cached tokens of slot b
    (no cache_batch_idx), as batched fp32 matmuls over chunks of rows (the CPU baseline's form of
    the same equation; equal to decode_ref up to fp32 summation order).  One row per chunk is
    the fastest on the host: a row's fp32 K/V transients (16 MiB at 4K x 8 x 128) are recycled by
    the allocator, while multi-row chunks page-fault fresh mappings every call (measured 0.15 vs
    0.9 s per Llama-3-8B layer on 8 cores).  q: [B, Hq, D]; k_cache/v_cache: [B, >= n, Hkv, D]."""
    batch, hq, d = q.shape
    hkv = k_cache.shape[2]
    group = hq // hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = torch.zeros(batch, hq, d, dtype=torch.float32)
    if n == 0:
        return out
    for b0 in range(0, batch, rows_per_chunk):
        b1 = min(batch, b0 + rows_per_chunk)
        k = k_cache[b0:b1, :n].float().permute(0, 2, 1, 3)            # [b, Hkv, n, D]
        v = v_cache[b0:b1, :n].float().permute(0, 2, 1, 3)
        qb = q[b0:b1].float().view(b1 - b0, hkv, group, d)            # head h -> kv head h // group
        s = torch.matmul(qb, k.transpose(-1, -2)) * scale             # [b, Hkv, group, n]
        p = torch.softmax(s, dim=-1)
        out[b0:b1] = torch.matmul(p, v).reshape(b1 - b0, hq, d)
    return out


def prefill_ref(q, k, v, causal=True, scale=None):
    """Self-attention of one request's Sq query rows over its Sk cached keys.

    q: [Sq, Hq, D]; k/v: [Sk, Hkv, D] (the slot's first Sk rows).  Returns fp32 [Sq, Hq, D].
    """
    sq, hq, d = q.shape
    sk, hkv = k.shape[0], k.shape[1]
    group = hq // hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    qf = q.float().permute(1, 0, 2)                               # [Hq, Sq, D]
    kf = k.float().permute(1, 0, 2).repeat_interleave(group, 0)   # [Hq, Sk, D]
    vf = v.float().permute(1, 0, 2).repeat_interleave(group, 0)
    out = torch.empty(hq, sq, d, dtype=torch.float32)
    chunk = 1024
    for i0 in range(0, sq, chunk):
        i1 = min(sq, i0 + chunk)
        s = torch.matmul(qf[:, i0:i1], kf.transpose(1, 2)) * scale
        if causal:
            qi = torch.arange(i0, i1).view(-1, 1) + (sk - sq)
            kj = torch.arange(sk).view(1, -1)
            s = s.masked_fill(kj > qi, float("-inf"))
        p = torch.softmax(s, dim=-1)
        p = torch.nan_to_num(p, nan=0.0)                          # fully-masked rows -> 0
        out[:, i0:i1] = torch.matmul(p, vf)
    return out.permute(1, 0, 2).contiguous()


def max_rel_err(out, ref) -> float:
    """North-star metric: max|o - o_ref| / max|o_ref|."""
    ref = ref.float()
    denom = ref.abs().max().item()
    return (out.float() - ref).abs().max().item() / max(denom, 1e-30)


def elem_rel_err(out, ref, eps: float = 1e-3) -> float:
    """Elementwise metric SURVEY §8(c) asks to report beside max_rel_err:
    max over elements of |o - o_ref| / (|o_ref| + eps).  It is dominated by near-zero reference
    elements (cancellation in the P·V sum), where a bf16-rounded P contributes an absolute error
    of order 2^-9 · mean|v|; the tests bound it separately from the north-star metric."""
    ref = ref.float()
    return ((out.float() - ref).abs() / (ref.abs() + eps)).max().item()


def err_report(out, ref) -> dict:
    """Both metrics plus the element count, for test logs and bench extras."""
    return {"max_rel_err": max_rel_err(out, ref), "elem_rel_err": elem_rel_err(out, ref), "elements": ref.numel()}


def rotary_ref(x, cos, sin, positions, interleaved=False):
    """Rotary embedding of x [B, H, D] at per-row positions [B] (fp32 result).

    cos/sin: [positions, rotary_dim/2]; dims >= rotary_dim pass through.  Non-interleaved =
    GPT-NeoX halves (x[i], x[i + rd/2]); interleaved = GPT-J pairs (x[2i], x[2i+1]).  This is
    flash-attn's apply_rotary_emb as flash_attn_with_kvcache applies it to q and k at
    cache_seqlens (the kernels the paper uses; not vendored in the reference).
    """
    x = x.float().clone()
    rd = 2 * cos.shape[1]
    c = cos.float()[positions.long()].unsqueeze(1)      # [B, 1, rd/2]
    s = sin.float()[positions.long()].unsqueeze(1)
    if interleaved:
        x1, x2 = x[..., 0:rd:2].clone(), x[..., 1:rd:2].clone()
        x[..., 0:rd:2] = x1 * c - x2 * s
        x[..., 1:rd:2] = x1 * s + x2 * c
    else:
        x1, x2 = x[..., : rd // 2].clone(), x[..., rd // 2: rd].clone()
        x[..., : rd // 2] = x1 * c - x2 * s
        x[..., rd // 2: rd] = x1 * s + x2 * c
    return x
