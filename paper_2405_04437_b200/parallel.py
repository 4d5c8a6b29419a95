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


def exchange_handles(blob: bytes, group=None) -> list[bytes]:
    """All-gather one fixed-size opaque handle per rank (rank order) over torch.distributed."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    got: list = [None] * world
    dist.all_gather_object(got, bytes(blob), group=group)
    if any(not isinstance(b, (bytes, bytearray)) or len(b) != len(blob) for b in got):
        raise RuntimeError("gather handle exchange: ranks disagree on the handle size")
    return [bytes(b) for b in got]


class HeadGather:
    """Fused output-head all-gather over NVLink peer memory.

    One per rank.  Holds this rank's two staging areas [max_batch, Hq_total, D] bf16 (launches
    alternate between them, so a peer's next launch never writes where a slow consumer still
    reads: csrc/gather.cu) plus the peer mappings of every other rank's buffer;
    `attention.decode_attention_gather` makes the decode kernel store each output row straight
    into all of them, and `wait()` orders the stream after every rank's rows landed and copies
    the full output into the caller's tensor (or the rank-local front buffer, `output()`).
    Every rank issues the same sequence of gathered launches, each followed by its `wait()` on
    the same stream.  Replaces `gather_heads` (NCCL all_gather) for the decode output; `create`
    is collective (CUDA IPC handles exchanged over torch.distributed), `local_group` simulates
    `world` ranks on one GPU in one process (tests, single-GPU boxes)."""

    def __init__(self, handle, rank: int, world: int, max_batch: int, hq_total: int, head_dim: int, device: int):
        self.handle = handle
        self.rank, self.world = rank, world
        self.max_batch, self.hq_total, self.head_dim = max_batch, hq_total, head_dim
        self.device = device
        self._view = None

    @staticmethod
    def _out_bytes(max_batch, hq_total, head_dim):
        if hq_total <= 0 or max_batch <= 0 or head_dim <= 0:
            raise ValueError("max_batch, hq_total and head_dim must be positive")
        return max_batch * hq_total * head_dim * 2

    @classmethod
    def create(cls, max_batch: int, hq_total: int, head_dim: int, group=None, device: int | None = None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from ._abi import IPC_HANDLE_BYTES, check, lib

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if hq_total % world:
            raise ValueError(f"{hq_total} query heads cannot be split over {world} ranks")
        dev = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        buf = (C.c_char * IPC_HANDLE_BYTES)()
        self, err = None, None
        try:
            check(lib().vattn_gather_create(dev, rank, world, cls._out_bytes(max_batch, hq_total, head_dim),
                                            C.byref(h), buf))
            self = cls(h, rank, world, max_batch, hq_total, head_dim, dev)
        except Exception as e:      # still take part in the exchange, so no peer blocks in it
            err = e
        # byte 0: this rank's setup status, then its IPC handle
        blobs = exchange_handles((b"\1" if err is None else b"\0") + bytes(buf), group)
        failed = [r for r, b in enumerate(blobs) if b[0] != 1]
        try:
            if err is not None:
                raise err
            if failed:
                raise RuntimeError(f"HeadGather: ranks {failed} failed to create their buffers")
            allh = (C.c_char * (IPC_HANDLE_BYTES * world)).from_buffer_copy(b"".join(b[1:] for b in blobs))
            check(lib().vattn_gather_open(h, allh))
        except Exception:
            if self is not None:
                self.close()
            raise
        return self

    @classmethod
    def local_group(cls, world: int, max_batch: int, hq_total: int, head_dim: int, device: int = 0):
        import ctypes as C

        from ._abi import check, lib

        if hq_total % world:
            raise ValueError(f"{hq_total} query heads cannot be split over {world} ranks")
        hs = (C.c_void_p * world)()
        check(lib().vattn_gather_create_local(device, world, cls._out_bytes(max_batch, hq_total, head_dim), hs))
        return [cls(C.c_void_p(hs[r]), r, world, max_batch, hq_total, head_dim, device) for r in range(world)]

    def output(self, batch: int | None = None):
        """Non-owning [batch, Hq_total, D] bf16 view of this rank's front buffer (what the last
        `wait()` without `out` delivered; rewritten by the next one on its stream)."""
        import ctypes as C

        import torch

        from ._abi import check, lib

        if self._view is None:
            ptr = C.c_uint64()
            check(lib().vattn_gather_output(self.handle, C.byref(ptr)))
            dev = torch.device("cuda", self.device)
            n = self._out_bytes(self.max_batch, self.hq_total, self.head_dim)
            storage = torch._C._construct_storage_from_data_pointer(ptr.value, dev, n)
            t = torch.empty(0, dtype=torch.bfloat16, device=dev)
            t.set_(storage, 0, (self.max_batch, self.hq_total, self.head_dim))
            self._view = t
        return self._view if batch is None else self._view[:batch]

    def wait(self, stream=None, out=None, batch: int | None = None):
        """Stream-ordered: wait for every rank's rows of the latest gathered launch, then copy
        the full [batch, Hq_total, D] output into `out` (default: the front buffer, returned as
        `output(batch)`).  batch 0 waits without copying and returns None."""
        import ctypes as C

        import torch

        from ._abi import check, lib

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if out is not None:
            if (out.dtype != torch.bfloat16 or not out.is_contiguous() or out.device.type != "cuda"
                    or out.device.index != self.device or out.dim() != 3
                    or tuple(out.shape[1:]) != (self.hq_total, self.head_dim)):
                raise ValueError(f"out must be a contiguous bf16 [B, {self.hq_total}, {self.head_dim}] tensor "
                                 f"on cuda:{self.device}")
            if batch is not None and batch != out.shape[0]:
                raise ValueError("batch disagrees with out.shape[0]")
            batch = out.shape[0]
        elif batch is None:
            batch = self.max_batch
        if not 0 <= batch <= self.max_batch:
            raise ValueError(f"batch {batch} outside [0, {self.max_batch}]")
        nbytes = batch * self.hq_total * self.head_dim * 2
        dst = None if out is None else C.c_void_p(out.data_ptr())
        check(lib().vattn_gather_wait(self.handle, dst, nbytes, C.c_void_p(s.cuda_stream)))
        if batch == 0:
            return None
        return out if out is not None else self.output(batch)

    def timed_out_ranks(self) -> list[int]:
        """Ranks whose rows a wait gave up on (a rank skipped a gathered launch); syncs."""
        import ctypes as C

        from ._abi import check, lib

        m = C.c_uint32()
        check(lib().vattn_gather_check(self.handle, C.byref(m)))
        return [r for r in range(self.world) if m.value >> r & 1]

    def close(self) -> None:
        if self.handle is not None:
            from ._abi import lib

            self._view = None
            lib().vattn_gather_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
