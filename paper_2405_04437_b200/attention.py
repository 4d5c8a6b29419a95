"""Attention entry points over the virtual KV cache (torch tensors only at this edge).

Semantics follow the paper's use of flash_attn_with_kvcache: q [B, Hq, D],
`cache_seqlens[b]` cached rows of slot `cache_batch_idx[b]`, GQA head h -> KV head h // (Hq/Hkv),
scale 1/sqrt(D) by default, bf16 in / fp32 accumulate / bf16 out.  Every op launches the sm_100a
kernels in libvattn.so on the current torch stream; there is no Python or CPU fallback — a
missing library or a non-CUDA tensor is an error.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import torch

from . import _abi
from ._abi import check, lib


def _stream(stream=None, device: int | None = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    # the raw handle of the current stream without building a torch.cuda.Stream object
    # (same value as torch.cuda.current_stream().cuda_stream, graph capture included; ~2 us less)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice() if device is None else device)


# Host-side shape checks of the manager-backed ops (no device->host copy): the kernels take head
# counts and head_dim from the manager's geometry and the batch from q, so a mismatched tensor
# would make them read or write past it (ADVICE r1 attention.py:103).
def _geom(mgr):
    g = mgr._g
    return g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim


def _on_mgr_device(mgr, *ts):
    for t in ts:
        if t is not None and (t.device.type != "cuda" or t.device.index != mgr.device):
            raise ValueError(f"tensors must live on the manager's device cuda:{mgr.device}, got {t.device}")


def _expect(t, shape, name):
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)} (manager geometry), got {tuple(t.shape)}")


def _check_out(out, shape, device):
    if (out.dtype != torch.bfloat16 or not out.is_contiguous() or tuple(out.shape) != tuple(shape)
            or out.device != device):
        raise ValueError(f"out must be a contiguous bf16 tensor of shape {tuple(shape)} on {device}")


def _check_rows(batch, seq, idx):
    if seq is None:
        raise ValueError("cache_seqlens is required")
    if seq.dim() != 1 or seq.numel() < batch:
        raise ValueError(f"cache_seqlens must be a 1-D tensor with at least {batch} entries")
    if idx is not None and (idx.dim() != 1 or idx.numel() < batch):
        raise ValueError(f"cache_batch_idx must be a 1-D tensor with at least {batch} entries")


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("attention ops take CUDA tensors (there is no CPU path)")


def _i32(t, name):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.dtype != torch.int32 or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA int32 tensor")
    return t.contiguous()


def _bf16(t, name):
    if t.dtype != torch.bfloat16:
        raise ValueError(f"{name} must be bfloat16")
    return t.contiguous()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


# Opt-in guard (VATTN_CHECK_BOUNDS=1): check on the host, before launch, that every cache row a
# kernel will touch is backed by a mapped page-group.  The kernels trust cache_seqlens (it lives
# on the device); a row past the mapped prefix of a slot would fault the GPU context instead of
# raising.  Costs one device->host copy of the index vectors per call, so it is off by default.
CHECK_BOUNDS = os.environ.get("VATTN_CHECK_BOUNDS", "0") not in ("", "0")


def check_bounds(mgr, cache_seqlens, cache_batch_idx=None, extra_rows: int = 0) -> None:
    """Raise ValueError unless rows [0, cache_seqlens[b] + extra_rows) of slot cache_batch_idx[b]
    are all backed (reference contract: only stepped lengths may be touched, manager.py:255-296)."""
    seq = cache_seqlens.tolist() if isinstance(cache_seqlens, torch.Tensor) else list(cache_seqlens)
    if cache_batch_idx is None:
        idx = list(range(len(seq)))
    else:
        idx = cache_batch_idx.tolist() if isinstance(cache_batch_idx, torch.Tensor) else list(cache_batch_idx)
    slots = mgr.slots
    for b, (n, r) in enumerate(zip(seq, idx)):
        if not 0 <= r < len(slots):
            raise ValueError(f"cache_batch_idx[{b}] = {r} is not a slot (max_batch {len(slots)})")
        backed = slots[r].mapped_groups * mgr.page_group_size // mgr.per_buffer_token_bytes
        if n < 0 or n + extra_rows > backed:
            raise ValueError(f"row {b}: slot {r} needs {n + extra_rows} tokens but only {backed} are mapped "
                             f"(call step() with the grown lengths first)")


# ------------------------------------------------------------------ manager-backed ops
def kv_append(mgr, layer: int, k_new, v_new, cache_seqlens, cache_batch_idx=None, stream=None,
              rotary_cos=None, rotary_sin=None, rotary_interleaved: bool = False):
    """Write k_new/v_new [B, T, Hkv, D] (or [B, Hkv, D] for one token) at rows
    cache_seqlens[b] .. +T of slot cache_batch_idx[b].  The rows must be backed (call
    mgr.step with the grown lengths first).  With rotary tables, k row i is cached rotated at
    position cache_seqlens[b] + i."""
    _need_cuda(k_new, v_new)
    _on_mgr_device(mgr, k_new, v_new)
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(1), v_new.unsqueeze(1)
    _, hkv, d = _geom(mgr)
    if k_new.dim() != 4:
        raise ValueError("k_new must be [B, T, Hkv, D] or [B, Hkv, D]")
    _expect(k_new, (k_new.shape[0], k_new.shape[1], hkv, d), "k_new")
    _expect(v_new, k_new.shape, "v_new")
    k_new, v_new = _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    _check_rows(k_new.shape[0], seq, idx)
    if CHECK_BOUNDS:
        check_bounds(mgr, seq, idx, extra_rows=k_new.shape[1])
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    st = C.c_void_p(_stream(stream, mgr.device))
    if rot is not None:
        check(lib().vattn_kv_append_rotary(mgr._h, layer, _ptr(k_new), _ptr(v_new), k_new.shape[0], k_new.shape[1],
                                           _ptr(seq), _ptr(idx), C.byref(rot), st))
        return
    check(lib().vattn_kv_append(mgr._h, layer, _ptr(k_new), _ptr(v_new), k_new.shape[0], k_new.shape[1],
                                _ptr(seq), _ptr(idx), st))


def decode_attention(mgr, layer: int, q, cache_seqlens, cache_batch_idx=None, softmax_scale=None,
                     out=None, num_splits: int = 0, stream=None):
    """o[b] = softmax(q[b] K[slot, :seqlen]ᵀ·scale) V[slot, :seqlen] for q [B, Hq, D]."""
    _need_cuda(q)
    _on_mgr_device(mgr, q)
    hq, _, d = _geom(mgr)
    _expect(q, (q.shape[0], hq, d), "q")
    q = _bf16(q, "q")
    if out is None:
        out = torch.empty_like(q)
    else:
        _check_out(out, q.shape, q.device)
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    _check_rows(q.shape[0], seq, idx)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    if CHECK_BOUNDS:
        check_bounds(mgr, seq, idx)
    check(lib().vattn_decode(mgr._h, layer, _ptr(q), _ptr(out), q.shape[0], _ptr(seq), _ptr(idx),
                             float(scale), int(num_splits), C.c_void_p(_stream(stream, mgr.device))))
    return out


def _check_decode_new(mgr, q, k_new, v_new):
    """q [B, Hq_local, D]; k_new / v_new [B, Hkv_local, D] (one new token per row)."""
    hq, hkv, d = _geom(mgr)
    _expect(q, (q.shape[0], hq, d), "q")
    if k_new is not None:
        _expect(k_new, (q.shape[0], hkv, d), "k_new")
        _expect(v_new, (q.shape[0], hkv, d), "v_new")


def _rotary(rotary_cos, rotary_sin, rotary_interleaved):
    """fp32 tables [positions, rotary_dim / 2] -> (descriptor, keep-alive tensors)."""
    if rotary_cos is None and rotary_sin is None:
        return None, None
    if rotary_cos is None or rotary_sin is None:
        raise ValueError("rotary_cos and rotary_sin go together")
    _need_cuda(rotary_cos, rotary_sin)
    if rotary_cos.shape != rotary_sin.shape or rotary_cos.dim() != 2:
        raise ValueError("rotary_cos / rotary_sin must both be [positions, rotary_dim / 2]")
    cos = rotary_cos.to(torch.float32).contiguous()
    sin = rotary_sin.to(torch.float32).contiguous()
    r = _abi.RotaryC()
    r.cos, r.sin = cos.data_ptr(), sin.data_ptr()
    r.rotary_dim, r.interleaved = 2 * cos.shape[1], int(bool(rotary_interleaved))
    return r, (cos, sin)


def decode_attention_append(mgr, layer: int, q, k_new, v_new, cache_seqlens, cache_batch_idx=None,
                            softmax_scale=None, out=None, num_splits: int = 0, stream=None,
                            rotary_cos=None, rotary_sin=None, rotary_interleaved: bool = False):
    """Fused KV-append + decode (flash_attn_with_kvcache k=/v=): k_new/v_new [B, Hkv, D] are
    written at row cache_seqlens[b] (the length before the token) and attended to, one launch.
    rotary_cos / rotary_sin [positions, rotary_dim / 2]: q and k_new are rotated at position
    cache_seqlens[b] first and k is cached rotated (flash-attn's rotary semantics)."""
    _need_cuda(q, k_new, v_new)
    _on_mgr_device(mgr, q, k_new, v_new)
    _check_decode_new(mgr, q, k_new, v_new)
    q, k_new, v_new = _bf16(q, "q"), _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    if out is None:
        out = torch.empty_like(q)
    else:
        _check_out(out, q.shape, q.device)
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    _check_rows(q.shape[0], seq, idx)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    if CHECK_BOUNDS:
        check_bounds(mgr, seq, idx, extra_rows=1)
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    st = C.c_void_p(_stream(stream, mgr.device))
    if rot is not None:
        check(lib().vattn_decode_append_rotary(mgr._h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out),
                                               q.shape[0], _ptr(seq), _ptr(idx), float(scale), int(num_splits),
                                               C.byref(rot), st))
        return out
    check(lib().vattn_decode_append(mgr._h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), q.shape[0],
                                    _ptr(seq), _ptr(idx), float(scale), int(num_splits), st))
    return out


def decode_attention_gather(mgr, layer: int, q, gather, cache_seqlens, cache_batch_idx=None, k_new=None,
                            v_new=None, softmax_scale=None, num_splits: int = 0, wait: bool = True, stream=None,
                            out=None):
    """Decode this rank's query heads q [B, Hq/G, D] (k_new/v_new given: fused append, as
    decode_attention_append) and all-gather the heads in the same kernel: every output row is
    stored over NVLink peer memory into each rank's staging area [B, Hq, D] at head offset
    rank*Hq/G.  With wait=True the stream then waits for all ranks' rows and the
    full output is copied to `out` (default: the gather's front buffer, `gather.output(B)`),
    which is returned; with wait=False call `gather.wait(stream, out)` before the next gathered
    launch and returns None."""
    _need_cuda(q)
    if (k_new is None) != (v_new is None):
        raise ValueError("k_new and v_new go together")
    _on_mgr_device(mgr, q, k_new, v_new)
    _check_decode_new(mgr, q, k_new, v_new)
    if q.shape[1] * gather.world != gather.hq_total or q.shape[2] != gather.head_dim:
        raise ValueError("q heads x gather world must equal the gather's Hq_total (and head_dim match)")
    if q.shape[0] > gather.max_batch:
        raise ValueError(f"batch {q.shape[0]} exceeds the gather's max_batch {gather.max_batch}")
    q = _bf16(q, "q")
    if k_new is not None:
        _need_cuda(k_new, v_new)
        k_new, v_new = _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    _check_rows(q.shape[0], seq, idx)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    if CHECK_BOUNDS:
        check_bounds(mgr, seq, idx, extra_rows=0 if k_new is None else 1)
    st = C.c_void_p(_stream(stream, mgr.device))
    check(lib().vattn_decode_gather(mgr._h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), gather.handle, q.shape[0],
                                    _ptr(seq), _ptr(idx), float(scale), int(num_splits), st))
    if not wait:
        return None
    return gather.wait(stream, out=out, batch=None if out is not None else q.shape[0])


def prefill_attention(mgr, layer: int, q, req_id: int, kv_len: int | None = None, causal=True,
                      softmax_scale=None, out=None, stream=None, rotary_cos=None, rotary_sin=None,
                      rotary_interleaved: bool = False):
    """Causal (bottom-right aligned) attention of q [S, Hq, D] over rows [0, kv_len) of slot
    req_id (default kv_len = S, i.e. the prompt just appended).  With rotary tables, query row i
    is rotated at position kv_len - S + i inside the kernel (append k with the same tables)."""
    _need_cuda(q)
    _on_mgr_device(mgr, q)
    hq, _, d = _geom(mgr)
    _expect(q, (q.shape[0], hq, d), "q")
    q = _bf16(q, "q")
    if out is None:
        out = torch.empty_like(q)
    else:
        _check_out(out, q.shape, q.device)
    kv_len = q.shape[0] if kv_len is None else kv_len
    if not 0 <= int(req_id) < mgr._g.max_batch:
        raise ValueError(f"req_id {req_id} is not a slot (max_batch {mgr._g.max_batch})")
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    if CHECK_BOUNDS:
        check_bounds(mgr, [kv_len], [req_id])
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    st = C.c_void_p(_stream(stream, mgr.device))
    if rot is not None:
        check(lib().vattn_prefill_rotary(mgr._h, layer, _ptr(q), _ptr(out), q.shape[0], int(req_id), int(kv_len),
                                         float(scale), int(bool(causal)), C.byref(rot), st))
        return out
    check(lib().vattn_prefill(mgr._h, layer, _ptr(q), _ptr(out), q.shape[0], int(req_id), int(kv_len),
                              float(scale), int(bool(causal)), st))
    return out


def _varlen_arrays(q, q_lens, req_ids, kv_lens):
    n = len(q_lens)
    if len(req_ids) != n or (kv_lens is not None and len(kv_lens) != n):
        raise ValueError("q_lens, req_ids and kv_lens must have one entry per request")
    kv_lens = list(q_lens) if kv_lens is None else list(kv_lens)
    starts, acc = [], 0
    for m in q_lens:
        starts.append(acc)
        acc += int(m)
    if acc != q.shape[0]:
        raise ValueError(f"packed q has {q.shape[0]} rows but q_lens sum to {acc}")
    arr = lambda xs: (C.c_int32 * max(1, n))(*[int(x) for x in xs])  # noqa: E731
    return n, arr(starts), arr(q_lens), arr(req_ids), arr(kv_lens)


def prefill_attention_varlen(mgr, layer: int, q, q_lens, req_ids, kv_lens=None, causal=True, softmax_scale=None,
                             out=None, stream=None):
    """Prefill of several requests in ONE launch (flash_attn_varlen_func-style): q [sum(q_lens),
    Hq, D] packs each request's query rows in order; request i attends (bottom-right causal)
    over rows [0, kv_lens[i]) of slot req_ids[i] (default kv_lens = q_lens)."""
    _need_cuda(q)
    _on_mgr_device(mgr, q)
    hq, _, d = _geom(mgr)
    _expect(q, (q.shape[0], hq, d), "q")
    q = _bf16(q, "q")
    if out is None:
        out = torch.empty_like(q)
    else:
        _check_out(out, q.shape, q.device)
    n, st, nq, sl, kl = _varlen_arrays(q, q_lens, req_ids, kv_lens)
    if any(not 0 <= int(r) < mgr._g.max_batch for r in req_ids):
        raise ValueError(f"req_ids must be slots in [0, {mgr._g.max_batch})")
    if CHECK_BOUNDS:
        check_bounds(mgr, list(kv_lens if kv_lens is not None else q_lens), list(req_ids))
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    check(lib().vattn_prefill_varlen(mgr._h, layer, _ptr(q), _ptr(out), n, st, nq, sl, kl, float(scale),
                                     int(bool(causal)), C.c_void_p(_stream(stream, mgr.device))))
    return out


def prefill_attention_varlen_raw(q, k_cache, v_cache, q_lens, slots, kv_lens=None, causal=True, softmax_scale=None,
                                 out=None, stream=None):
    desc = cache_desc(k_cache, v_cache)
    q = _bf16(q, "q")
    out = torch.empty_like(q) if out is None else out
    n, st, nq, sl, kl = _varlen_arrays(q, q_lens, slots, kv_lens)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(q.shape[-1])
    check(lib().vattn_prefill_varlen_raw(C.byref(desc), _ptr(q), _ptr(out), q.shape[1], n, st, nq, sl, kl,
                                         float(scale), int(bool(causal)), C.c_void_p(_stream(stream))))
    return out


# ------------------------------------------------------------------ standalone ops
def cache_desc(k_cache, v_cache) -> _abi.CacheDesc:
    """Descriptor of caller-owned token-major caches [slots, tokens, Hkv, D] (any slot/token
    strides, rows contiguous)."""
    _need_cuda(k_cache, v_cache)
    if k_cache.dtype != torch.bfloat16 or v_cache.dtype != torch.bfloat16:
        raise ValueError("caches must be bfloat16")
    if k_cache.shape != v_cache.shape or k_cache.stride() != v_cache.stride():
        raise ValueError("K and V caches must share shape and strides")
    n, L, h, d = k_cache.shape
    if k_cache.stride(3) != 1 or k_cache.stride(2) != d:
        raise ValueError("each token row [Hkv, D] must be contiguous")
    desc = _abi.CacheDesc()
    desc.k_base, desc.v_base = k_cache.data_ptr(), v_cache.data_ptr()
    desc.slot_stride_bytes = k_cache.stride(0) * 2
    desc.token_stride_bytes = k_cache.stride(1) * 2
    desc.slot_tokens, desc.n_slots, desc.n_kv_heads, desc.head_dim = L, n, h, d
    return desc


def kv_append_raw(k_cache, v_cache, k_new, v_new, cache_seqlens, cache_batch_idx=None, stream=None,
                  rotary_cos=None, rotary_sin=None, rotary_interleaved: bool = False):
    desc = cache_desc(k_cache, v_cache)
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(1), v_new.unsqueeze(1)
    k_new, v_new = _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    if rot is not None:
        check(lib().vattn_kv_append_rotary_raw(C.byref(desc), _ptr(k_new), _ptr(v_new), k_new.shape[0],
                                               k_new.shape[1], _ptr(seq), _ptr(idx), C.byref(rot),
                                               C.c_void_p(_stream(stream))))
        return
    check(lib().vattn_kv_append_raw(C.byref(desc), _ptr(k_new), _ptr(v_new), k_new.shape[0], k_new.shape[1],
                                    _ptr(seq), _ptr(idx), C.c_void_p(_stream(stream))))


_ws_cache: dict = {}
_ws_retired: list = []


def _workspace(device, nbytes, stream=None):
    """Split-K workspace of the raw ops, one per (device, launching stream): two streams never
    share partials.  A grown workspace retires the old one without freeing it, since a CUDA
    graph may have captured its address."""
    key = (device, _stream(stream))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:
            _ws_retired.append(ws)
        ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def decode_attention_raw(q, k_cache, v_cache, cache_seqlens, cache_batch_idx=None, softmax_scale=None,
                         out=None, num_splits: int = 0, stream=None):
    desc = cache_desc(k_cache, v_cache)
    q = _bf16(q, "q")
    out = torch.empty_like(q) if out is None else out
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    b, hq, d = q.shape
    nbytes = lib().vattn_decode_workspace_bytes(b, hq, d, 0)
    ws = _workspace(q.device, nbytes, stream)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    check(lib().vattn_decode_raw(C.byref(desc), _ptr(q), _ptr(out), b, hq, _ptr(seq), _ptr(idx), float(scale),
                                 int(num_splits), _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
    return out


def decode_attention_append_raw(q, k_cache, v_cache, k_new, v_new, cache_seqlens, cache_batch_idx=None,
                                softmax_scale=None, out=None, num_splits: int = 0, stream=None,
                                rotary_cos=None, rotary_sin=None, rotary_interleaved: bool = False):
    desc = cache_desc(k_cache, v_cache)
    q, k_new, v_new = _bf16(q, "q"), _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    out = torch.empty_like(q) if out is None else out
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    b, hq, d = q.shape
    ws = _workspace(q.device, lib().vattn_decode_workspace_bytes(b, hq, d, 0), stream)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    if rot is not None:
        check(lib().vattn_decode_append_rotary_raw(C.byref(desc), _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), b,
                                                   hq, _ptr(seq), _ptr(idx), float(scale), int(num_splits),
                                                   C.byref(rot), _ptr(ws), ws.numel(), C.c_void_p(_stream(stream))))
        return out
    check(lib().vattn_decode_append_raw(C.byref(desc), _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), b, hq,
                                        _ptr(seq), _ptr(idx), float(scale), int(num_splits), _ptr(ws), ws.numel(),
                                        C.c_void_p(_stream(stream))))
    return out


def decode_attention_gather_raw(q, k_cache, v_cache, gather, cache_seqlens, cache_batch_idx=None, k_new=None,
                                v_new=None, softmax_scale=None, num_splits: int = 0, wait: bool = True,
                                stream=None, out=None):
    """decode_attention_gather on caller-owned caches (see cache_desc)."""
    desc = cache_desc(k_cache, v_cache)
    q = _bf16(q, "q")
    if k_new is not None:
        k_new, v_new = _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    seq = _i32(cache_seqlens, "cache_seqlens")
    idx = _i32(cache_batch_idx, "cache_batch_idx")
    b, hq, d = q.shape
    ws = _workspace(q.device, lib().vattn_decode_workspace_bytes(b, hq, d, 0), stream)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    check(lib().vattn_decode_gather_raw(C.byref(desc), _ptr(q), _ptr(k_new), _ptr(v_new), gather.handle, b, hq,
                                        _ptr(seq), _ptr(idx), float(scale), int(num_splits), _ptr(ws), ws.numel(),
                                        C.c_void_p(_stream(stream))))
    if not wait:
        return None
    return gather.wait(stream, out=out, batch=None if out is not None else b)


def decode_attention_paged(q, k_pool, v_pool, block_table, seqlens, softmax_scale=None, out=None,
                           num_splits: int = 0, stream=None):
    """PagedAttention-layout comparison kernel: pools [num_blocks, block_size, Hkv, D],
    block_table [B, max_blocks] int32 (PAPER.md:602 block sizes 16 / 256)."""
    _need_cuda(q, k_pool, v_pool)
    q = _bf16(q, "q")
    k_pool, v_pool = _bf16(k_pool, "k_pool"), _bf16(v_pool, "v_pool")
    out = torch.empty_like(q) if out is None else out
    bt = _i32(block_table, "block_table")
    seq = _i32(seqlens, "seqlens")
    b, hq, d = q.shape
    nb, bs, hkv, _ = k_pool.shape
    nbytes = lib().vattn_decode_workspace_bytes(b, hq, d, 0)
    ws = _workspace(q.device, nbytes, stream)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    check(lib().vattn_decode_paged(_ptr(q), _ptr(k_pool), _ptr(v_pool), nb, bs, hkv, d, _ptr(bt), bt.shape[1],
                                   _ptr(out), b, hq, _ptr(seq), float(scale), int(num_splits), _ptr(ws),
                                   ws.numel(), C.c_void_p(_stream(stream))))
    return out


def decode_num_splits(batch: int, n_kv_heads: int, max_seqlen: int) -> int:
    return lib().vattn_decode_num_splits(batch, n_kv_heads, max_seqlen)


def decode_kernel_name(batch: int, n_kv_heads: int, max_seqlen: int, num_splits: int = 0,
                       head_dim: int = 128) -> str:
    """Kernel variant a contiguous decode launch of this shape runs (measurement labels)."""
    buf = C.create_string_buffer(128)
    if lib().vattn_decode_kernel_name(batch, n_kv_heads, max_seqlen, num_splits, head_dim, buf, 128) < 0:
        raise RuntimeError("vattn_decode_kernel_name failed")
    return buf.value.decode()


def prefill_attention_raw(q, k_cache, v_cache, req_slot: int, kv_len: int, causal=True,
                          softmax_scale=None, out=None, stream=None, rotary_cos=None, rotary_sin=None,
                          rotary_interleaved: bool = False):
    desc = cache_desc(k_cache, v_cache)
    q = _bf16(q, "q")
    out = torch.empty_like(q) if out is None else out
    n_q, hq, d = q.shape
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    rot, _keep = _rotary(rotary_cos, rotary_sin, rotary_interleaved)
    if rot is not None:
        check(lib().vattn_prefill_rotary_raw(C.byref(desc), _ptr(q), _ptr(out), n_q, hq, int(req_slot), int(kv_len),
                                             float(scale), int(bool(causal)), C.byref(rot),
                                             C.c_void_p(_stream(stream))))
        return out
    check(lib().vattn_prefill_raw(C.byref(desc), _ptr(q), _ptr(out), n_q, hq, int(req_slot), int(kv_len),
                                  float(scale), int(bool(causal)), C.c_void_p(_stream(stream))))
    return out


def prefill_attention_paged(q, k_pool, v_pool, block_table, kv_len: int, causal=True, softmax_scale=None,
                            out=None, stream=None):
    """PagedAttention-layout comparison for prefill: the same tcgen05 kernel, K/V tiles gathered
    block by block through `block_table` [max_blocks] (one request).  Pool rows past kv_len in the
    last block must be finite (they are multiplied by zero)."""
    _need_cuda(q, k_pool, v_pool)
    q, k_pool, v_pool = _bf16(q, "q"), _bf16(k_pool, "k_pool"), _bf16(v_pool, "v_pool")
    out = torch.empty_like(q) if out is None else out
    bt = _i32(block_table, "block_table")
    n_q, hq, d = q.shape
    nb, bs, hkv, _ = k_pool.shape
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    check(lib().vattn_prefill_paged(_ptr(q), _ptr(k_pool), _ptr(v_pool), nb, bs, hkv, d, _ptr(bt), int(kv_len),
                                    _ptr(out), n_q, hq, float(scale), int(bool(causal)), C.c_void_p(_stream(stream))))
    return out


def kv_append_paged(k_pool, v_pool, k_new, v_new, block_table, cache_seqlens, stream=None):
    """PagedAttention-layout append: k_new/v_new [B, T, Hkv, D] (or [B, Hkv, D]) at rows
    cache_seqlens[b] + i, located through block_table [B, max_blocks]."""
    _need_cuda(k_pool, v_pool, k_new, v_new)
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(1), v_new.unsqueeze(1)
    k_new, v_new = _bf16(k_new, "k_new"), _bf16(v_new, "v_new")
    bt = _i32(block_table, "block_table")
    seq = _i32(cache_seqlens, "cache_seqlens")
    nb, bs, hkv, d = k_pool.shape
    check(lib().vattn_kv_append_paged(_ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool), bs, hkv, d, _ptr(bt),
                                      bt.shape[-1], k_new.shape[0], k_new.shape[1], _ptr(seq),
                                      C.c_void_p(_stream(stream))))
