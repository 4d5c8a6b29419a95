"""KV-head sharding across GPUs: one process per GPU, each running an independent
allocator + kernels over its heads; the only collective is the optional output-head all-gather.

Rank g owns KV heads [g·Hkv/G, (g+1)·Hkv/G) and the matching query heads (GQA groups stay whole).
Every rank's bookkeeping equals the reference KVCacheManager over geometry.with_tp(G)
(geometry.py:90-98, "all workers behave the same").
"""

from __future__ import annotations

from .geometry import ModelGeometry, as_geometry


def shard_geometry(geometry, world: int) -> ModelGeometry:
    g = as_geometry(geometry)
    if g.kv_heads_total % world:
        raise ValueError(f"{g.kv_heads_total} KV heads cannot be split over {world} GPUs")
    return g.with_tp(world)


def head_ranges(geometry, rank: int, world: int):
    """((kv_lo, kv_hi), (q_lo, q_hi)) owned by `rank`."""
    g = as_geometry(geometry)
    kv = g.kv_heads_total // world
    q = g.q_heads_total // world
    return (rank * kv, (rank + 1) * kv), (rank * q, (rank + 1) * q)


def shard_heads(x, geometry, rank: int, world: int, dim: int = -2, kind: str = "q"):
    """Slice a full-head tensor ([..., H, D]) down to this rank's heads."""
    (klo, khi), (qlo, qhi) = head_ranges(geometry, rank, world)
    lo, hi = (qlo, qhi) if kind == "q" else (klo, khi)
    return x.narrow(dim, lo, hi - lo)


def gather_heads(local, group=None, dim: int = -2):
    """All-gather every rank's [B, Hq/G, D] output into [B, Hq, D] (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return local
    d = dim % local.dim()
    moved = local.movedim(d, 0).contiguous()
    out = torch.empty((world * moved.shape[0],) + tuple(moved.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, moved, group=group)
    return out.movedim(0, d)
