"""Sizing math for the KV cache (the part of kvsim/geometry.py the hot path consumes).

Exact integer arithmetic, same definitions as the reference:
  per_token_layer_bytes  geometry.py:100-103   (H/TP)·D·P
  prefill_page_groups    geometry.py:177-183   ceil(size / t)
  block_size_tokens      geometry.py:150-158   t // per_token_layer_bytes
The build adds `n_q_heads_total` because the attention kernels need it.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, replace

KIB = 1024
MB2 = 2 * KIB * KIB
PAGE_GROUP_SIZES = (64 * KIB, 128 * KIB, 256 * KIB, MB2)


@dataclass(frozen=True)
class ModelGeometry:
    n_layers: int
    kv_heads_total: int
    head_dim: int
    bytes_per_elem: int
    max_context: int
    max_batch: int
    tp_degree: int = 1
    n_q_heads_total: int = 0   # 0 = no GQA (= kv_heads_total)

    def __post_init__(self) -> None:
        for name in ("n_layers", "kv_heads_total", "head_dim", "bytes_per_elem", "tp_degree"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")
        for name in ("max_context", "max_batch"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0, got {getattr(self, name)}")
        if self.kv_heads_total % self.tp_degree:
            raise ValueError("kv_heads_total must be divisible by tp_degree")
        hq = self.q_heads_total
        if hq % self.kv_heads_total or hq % self.tp_degree:
            raise ValueError("n_q_heads_total must be a multiple of kv_heads_total and tp_degree")

    @property
    def q_heads_total(self) -> int:
        return self.n_q_heads_total or self.kv_heads_total

    @property
    def kv_heads_per_worker(self) -> int:
        return self.kv_heads_total // self.tp_degree

    @property
    def q_heads_per_worker(self) -> int:
        return self.q_heads_total // self.tp_degree

    @property
    def group_size(self) -> int:
        return self.q_heads_total // self.kv_heads_total

    @property
    def per_token_layer_bytes(self) -> int:
        return self.kv_heads_per_worker * self.head_dim * self.bytes_per_elem

    def with_tp(self, tp_degree: int) -> "ModelGeometry":
        return replace(self, tp_degree=tp_degree)

    def to_dict(self) -> dict:
        return asdict(self)


def as_geometry(g) -> ModelGeometry:
    """Accept this package's ModelGeometry or any object with the reference's fields."""
    if isinstance(g, ModelGeometry):
        return g
    return ModelGeometry(
        n_layers=g.n_layers, kv_heads_total=g.kv_heads_total, head_dim=g.head_dim,
        bytes_per_elem=g.bytes_per_elem, max_context=g.max_context, max_batch=g.max_batch,
        tp_degree=getattr(g, "tp_degree", 1), n_q_heads_total=getattr(g, "n_q_heads_total", 0))


def prefill_page_groups(size_bytes: int, page_group_bytes: int) -> int:
    if size_bytes < 0:
        raise ValueError(f"size_bytes must be >= 0, got {size_bytes}")
    if page_group_bytes < 1:
        raise ValueError(f"page_group_bytes must be >= 1, got {page_group_bytes}")
    return -(-size_bytes // page_group_bytes)


def block_size_tokens(g: ModelGeometry, page_group_bytes: int) -> int:
    if page_group_bytes < g.per_token_layer_bytes:
        raise ValueError("page-group smaller than one token's per-layer cache")
    return page_group_bytes // g.per_token_layer_bytes


# BASELINE.json configurations (SURVEY §8 notation)
def tiny() -> ModelGeometry:
    return ModelGeometry(1, 2, 64, 2, max_context=512, max_batch=2, n_q_heads_total=8)


def llama3_8b(max_context: int = 8192, max_batch: int = 64) -> ModelGeometry:
    return ModelGeometry(32, 8, 128, 2, max_context=max_context, max_batch=max_batch,
                         n_q_heads_total=32)


def yi_6b(max_context: int = 16384, max_batch: int = 1) -> ModelGeometry:
    return ModelGeometry(32, 4, 128, 2, max_context=max_context, max_batch=max_batch,
                         n_q_heads_total=32)


def yi_34b(max_context: int = 8192, max_batch: int = 128, tp: int = 1) -> ModelGeometry:
    return ModelGeometry(60, 8, 128, 2, max_context=max_context, max_batch=max_batch,
                         tp_degree=tp, n_q_heads_total=56)
