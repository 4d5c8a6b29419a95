"""KVCacheManager — drop-in for the reference allocator (kvsim/manager.py:84-372) backed by the
C++ core in libvattn.so.

Same constructor (`KVCacheManager(geometry, ManagerConfig)`), same methods, same return types,
same exceptions, and the same introspection surface the reference tests read (`slots`,
`buffers`, `eager_slot`, `vmm.pool.*`, `vmm.calls`, `vmm.total_charged_us()` …).  What changes
is underneath: with the CUDA backend every page-group map/unmap is a real 2 MiB
cuMemMap/cuMemSetAccess/cuMemUnmap on a cuMemAddressReserve'd virtual tensor, and the
§6.1 overlap / eager / reclaim work can run on a real background thread (`bg_submit` /
`bg_wait`).  `k_cache(layer)` / `v_cache(layer)` are the virtual tensors Table 3 `init` returns.

Backends: "cuda" (default) or "shadow" (bookkeeping only — the reference's own semantics, no
device; selected explicitly, e.g. for CPU parity tests, or via VATTN_BACKEND=shadow).
"""

from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

from . import _abi
from ._abi import check, lib
from .errors import BatchFullError, DoubleFreeError  # noqa: F401  (re-export)
from .geometry import ModelGeometry, as_geometry, prefill_page_groups

DEFAULT_POOL_BYTES = 80 * 1024 ** 3   # vmm.py:23


class Phase(enum.Enum):           # manager.py:36-39
    INACTIVE = "inactive"
    PREFILL = "prefill"
    DECODE = "decode"


_PHASES = (Phase.INACTIVE, Phase.PREFILL, Phase.DECODE)


@dataclass
class ManagerConfig:              # manager.py:42-63
    page_group_size: int
    pool_bytes: int = DEFAULT_POOL_BYTES
    reclaim_threshold: float = 0.10
    eager_groups: int = 0
    sliced: bool = False
    pre_create_fraction: float = 1.0
    latency_model: object | None = None

    def __post_init__(self) -> None:
        if not 0.0 <= self.reclaim_threshold <= 1.0:
            raise ValueError("reclaim_threshold must be in [0, 1]")
        if not 0.0 <= self.pre_create_fraction <= 1.0:
            raise ValueError("pre_create_fraction must be in [0, 1]")
        if self.eager_groups < 0:
            raise ValueError("eager_groups must be >= 0")


@dataclass
class RequestSlot:                # manager.py:66-75 (a read-only snapshot here)
    req_id: int
    active: bool = False
    context_len: int = 0
    mapped_groups: int = 0
    phase: Phase = Phase.INACTIVE
    freed_seq: int = 0


@dataclass
class StepResult:                 # manager.py:78-81 (+ measured fields)
    ok: bool
    sync_us: float = 0.0
    wall_us: float = 0.0
    bg_wait_us: float = 0.0


@dataclass
class BackgroundResult:
    plan_us: float
    eager_us: float
    reclaim_us: float
    reclaimed_groups: int
    bg_wall_us: float
    waited_us: float


@dataclass
class IterationResult:
    ok: bool
    deferred: bool
    sync_us: float
    eager_us: float
    reclaim_us: float
    reclaimed_groups: int
    bg_wait_us: float
    sync_bg_wall_us: float
    wall_us: float


class _Pool:
    """PhysicalPool view (vmm.py:102-127)."""

    def __init__(self, mgr: "KVCacheManager"):
        self._m = mgr

    def _c(self):
        return self._m._counters()

    capacity = property(lambda self: self._c().capacity)
    page_group_size = property(lambda self: self._c().page_group_size)
    created = property(lambda self: self._c().created)
    mapped = property(lambda self: self._c().mapped)
    created_bytes = property(lambda self: self._c().created * self._c().page_group_size)
    mapped_bytes = property(lambda self: self._c().mapped * self._c().page_group_size)
    free_bytes = property(lambda self: self._c().capacity - self._c().created * self._c().page_group_size)
    available_bytes = property(lambda self: self._c().capacity - self._c().mapped * self._c().page_group_size)


class _Vmm:
    """VmmDevice view (vmm.py:150-302): counters, per-API calls and modelled ledger."""

    def __init__(self, mgr: "KVCacheManager"):
        self._m = mgr
        self.pool = _Pool(mgr)

    def _stats(self):
        n = lib().vattn_api_count()
        calls = (C.c_int64 * n)()
        ledger = (C.c_double * n)()
        order = (C.c_int32 * n)()
        n_order = C.c_int32()
        check(lib().vattn_api_stats(self._m._h, calls, ledger, order, C.byref(n_order)))
        names = _abi.api_names()
        return [(names[order[i]], calls[order[i]], ledger[order[i]]) for i in range(n_order.value)]

    @property
    def calls(self) -> dict:
        return {name: c for name, c, _ in self._stats()}

    @property
    def ledger_us(self) -> dict:
        return {name: us for name, _, us in self._stats()}

    def total_charged_us(self) -> float:
        return self._m._counters().charged_us

    @property
    def total_mapped_bytes(self) -> int:
        return self._m._counters().total_mapped_bytes

    @property
    def precreated_available(self) -> int:
        return self._m._counters().precreated


class _Buffer:
    """VirtualKVBuffer view (vmm.py:141-147) with its device address."""

    def __init__(self, mgr: "KVCacheManager", buffer_id: int, size: int):
        self._m, self.buffer_id, self.size = mgr, buffer_id, size

    @property
    def mappings(self) -> dict:
        n = C.c_int64()
        check(lib().vattn_buffer_mappings(self._m._h, self.buffer_id, None, None, 0, C.byref(n)))
        offs = (C.c_int64 * max(1, n.value))()
        hids = (C.c_int64 * max(1, n.value))()
        check(lib().vattn_buffer_mappings(self._m._h, self.buffer_id, offs, hids, n.value, C.byref(n)))
        return {offs[i]: hids[i] for i in range(n.value)}

    @property
    def device_ptr(self) -> int:
        p = C.c_uint64()
        check(lib().vattn_buffer_base(self._m._h, self.buffer_id, C.byref(p)))
        return p.value


def _latency_entries(model):
    if model is None:
        return None, 0
    table = getattr(model, "costs_us", model)   # kvsim LatencyModel or a plain dict
    rows = [(str(api), int(size), float(us)) for api, sizes in table.items() for size, us in sizes.items()]
    arr = (_abi.LatencyEntry * len(rows))()
    keep = []
    for i, (api, size, us) in enumerate(rows):
        b = api.encode()
        keep.append(b)
        arr[i].api, arr[i].page_group_bytes, arr[i].us = b, size, us
    return (arr, keep), len(rows)


class KVCacheManager:
    """vAttention KV-cache manager (Table 3 API: init / alloc_reqid / free_reqid / step)."""

    def __init__(self, geometry, config, *, backend: str | None = None, device: int | None = None,
                 log_events: bool | None = None, release_physical: bool = False,
                 batch_set_access: bool = True, prefetch_tokens: int = 0, prefetch_slots: int = 0,
                 prefetch_slot_tokens: int = 0, lazy_unmap: bool = False, phys_chunk_groups: int = 1):
        g = as_geometry(geometry)
        if g.max_batch < 1:
            raise ValueError("geometry.max_batch must be >= 1 to serve requests")
        backend = backend or os.environ.get("VATTN_BACKEND", "cuda")
        if backend not in ("cuda", "shadow"):
            raise ValueError(f"backend must be 'cuda' or 'shadow', got {backend!r}")
        if device is None:
            device = 0
            if backend == "cuda":
                import torch
                device = torch.cuda.current_device()
        self.geometry = geometry
        self.config = config
        self.backend = backend
        self.device = device
        cfg = _abi.Config()
        cfg.n_layers, cfg.kv_heads_total, cfg.head_dim = g.n_layers, g.kv_heads_total, g.head_dim
        cfg.bytes_per_elem, cfg.tp_degree, cfg.n_q_heads_total = g.bytes_per_elem, g.tp_degree, g.n_q_heads_total
        cfg.max_context, cfg.max_batch = g.max_context, g.max_batch
        cfg.page_group_size = int(config.page_group_size)
        cfg.pool_bytes = int(config.pool_bytes)
        cfg.reclaim_threshold = float(config.reclaim_threshold)
        cfg.pre_create_fraction = float(config.pre_create_fraction)
        cfg.eager_groups = int(config.eager_groups)
        cfg.sliced = int(bool(config.sliced))
        cfg.backend = 1 if backend == "cuda" else 0
        cfg.device = int(device)
        cfg.release_physical = int(release_physical)
        cfg.log_events = int(backend == "shadow" if log_events is None else log_events)
        cfg.batch_set_access = int(batch_set_access)
        cfg.prefetch_tokens = int(prefetch_tokens)
        cfg.prefetch_slots = int(prefetch_slots)
        cfg.prefetch_slot_tokens = int(prefetch_slot_tokens)
        cfg.lazy_unmap = int(bool(lazy_unmap))
        if int(phys_chunk_groups) < 1:
            raise ValueError("phys_chunk_groups must be >= 1")
        cfg.phys_chunk_groups = int(phys_chunk_groups)
        lat, n_lat = _latency_entries(getattr(config, "latency_model", None))
        if lat is not None:
            cfg.latency, cfg.n_latency = C.cast(lat[0], C.POINTER(_abi.LatencyEntry)), n_lat
        h = C.c_void_p()
        check(lib().vattn_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._g = g
        c = self._counters()
        self.page_group_size = c.page_group_size
        self.buffer_count = c.buffer_count
        self.per_buffer_token_bytes = c.per_buffer_token_bytes
        self.groups_per_slot = c.groups_per_slot
        self.slot_stride = c.slot_stride
        self.init_us = c.init_us
        self.init_wall_us = c.init_wall_us
        self.vmm = _Vmm(self)
        self.buffers = [_Buffer(self, i, c.buffer_size) for i in range(c.buffer_count)]
        self._n = g.max_batch
        self._seq = (C.c_int64 * self._n)()
        self._last_plan = None
        self._views = {}

    # -- lifetime --------------------------------------------------------------------------
    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        self._views = {}
        if h:
            check(lib().vattn_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _counters(self) -> _abi.Counters:
        c = _abi.Counters()
        check(lib().vattn_counters_get(self._h, C.byref(c)))
        return c

    # -- reference sizing helpers (manager.py:134-158) ---------------------------------------
    def groups_required(self, seq_len: int) -> int:
        return prefill_page_groups(seq_len * self.per_buffer_token_bytes, self.page_group_size)

    def slot_offset(self, req_id: int, group_index: int) -> int:
        return req_id * self.slot_stride + group_index * self.page_group_size

    @property
    def slots(self) -> list[RequestSlot]:
        raw = (C.c_int64 * (5 * self._n))()
        check(lib().vattn_slot_state(self._h, raw, self._n))
        return [RequestSlot(r, bool(raw[5 * r]), raw[5 * r + 1], raw[5 * r + 2], _PHASES[raw[5 * r + 3]],
                            raw[5 * r + 4]) for r in range(self._n)]

    @property
    def eager_slot(self):
        e = self._counters().eager_slot
        return None if e < 0 else e

    def slot_committed_bytes(self, req_id: int) -> int:
        return self.slots[req_id].mapped_groups * self.buffer_count * self.page_group_size

    def slot_used_bytes(self, req_id: int) -> int:
        return self.slots[req_id].context_len * self.per_buffer_token_bytes * self.buffer_count

    def committed_bytes(self) -> int:
        c = self._counters()
        return c.mapped * c.page_group_size

    def deferred_groups(self) -> int:
        return sum(s.mapped_groups for s in self.slots if not s.active)

    def free_slot_available(self) -> bool:
        return any(not s.active for s in self.slots)

    # -- Table 3 API ----------------------------------------------------------------------------
    def alloc_reqid(self) -> int:
        r = C.c_int32()
        check(lib().vattn_alloc_reqid(self._h, C.byref(r)))
        return r.value

    def free_reqid(self, req_id: int) -> None:
        check(lib().vattn_free_reqid(self._h, int(req_id)))

    def _fill_seq(self, seq_lens):
        if len(seq_lens) != self._n:
            raise ValueError(f"expected {self._n} sequence lengths, got {len(seq_lens)}")
        buf = self._seq
        for i, s in enumerate(seq_lens):
            buf[i] = int(s)
        return buf

    def step(self, seq_lens) -> StepResult:
        buf = self._fill_seq(seq_lens)
        out = _abi.StepResultC()
        check(lib().vattn_step(self._h, buf, self._n, C.byref(out)))
        return StepResult(bool(out.ok), out.sync_us, out.wall_us, out.bg_wait_us)

    # -- §6.1 optimisations ----------------------------------------------------------------------
    def plan_overlap(self, next_seq_lens) -> list[tuple[int, int, int]]:
        buf = self._fill_seq(next_seq_lens)
        n = C.c_int64()
        check(lib().vattn_plan_overlap(self._h, buf, self._n, C.byref(n)))
        raw = (C.c_int64 * max(1, 3 * n.value))()
        check(lib().vattn_plan_fetch(self._h, raw, n.value))
        plan = [(raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]) for i in range(n.value)]
        self._last_plan = plan
        return plan

    @staticmethod
    def _plan_array(plan):
        flat = (C.c_int64 * max(1, 3 * len(plan)))()
        for i, (r, b, o) in enumerate(plan):
            flat[3 * i], flat[3 * i + 1], flat[3 * i + 2] = int(r), int(b), int(o)
        return flat

    def execute_plan(self, plan) -> float:
        us = C.c_double()
        check(lib().vattn_execute_plan(self._h, self._plan_array(plan), len(plan), C.byref(us)))
        return us.value

    def eager_prepare(self, k_groups: int | None = None) -> float:
        us = C.c_double()
        check(lib().vattn_eager_prepare(self._h, -1 if k_groups is None else int(k_groups), C.byref(us)))
        return us.value

    def reclaim(self) -> tuple[int, float]:
        f, us = C.c_int64(), C.c_double()
        check(lib().vattn_reclaim(self._h, C.byref(f), C.byref(us)))
        return f.value, us.value

    def _reclaim_until(self, target_available_bytes: int) -> tuple[int, float]:
        f, us = C.c_int64(), C.c_double()
        check(lib().vattn_reclaim_until(self._h, int(target_available_bytes), C.byref(f), C.byref(us)))
        return f.value, us.value

    # -- the background mapping thread (§6.1.1/§6.1.2; simulator.py:199-203 order) ----------------
    def bg_submit(self, plan=None, *, execute_plan: bool = True, eager: bool = False,
                  reclaim: bool = False, eager_k: int | None = None, credit: bool = False,
                  prefetch: bool = False) -> None:
        """Queue execute_plan → eager_prepare → reclaim on the background thread.  Every other
        call joins the queue first (free_reqid only waits for queued eager/reclaim), so state is
        never mutated concurrently.  credit=True: the plan runs ahead of the next admission;
        alloc_reqid then ranks slots as if it had run after (the reference's order)."""
        flags = ((_abi.BG_EXECUTE_PLAN if execute_plan else 0) | (_abi.BG_EAGER if eager else 0)
                 | (_abi.BG_RECLAIM if reclaim else 0) | (_abi.BG_CREDIT if credit else 0)
                 | (_abi.BG_PREFETCH if prefetch else 0))
        if plan is None or plan is self._last_plan:
            arr, n = None, 0
        else:
            arr, n = self._plan_array(plan), len(plan)
        check(lib().vattn_bg_submit(self._h, arr, n, flags, -1 if eager_k is None else int(eager_k)))

    def iteration_step(self, seq_lens, *, eager: bool = True, reclaim: bool = True, defer: bool = True,
                       eager_k: int | None = None) -> "IterationResult":
        """One serving iteration's allocation work in the reference order (simulator.py:414-426):
        join the background queue, eager_prepare + reclaim (deferred behind step onto the
        background thread when provably equivalent), then step."""
        buf = self._fill_seq(seq_lens)
        flags = ((_abi.BG_EAGER if eager else 0) | (_abi.BG_RECLAIM if reclaim else 0)
                 | (_abi.ITER_DEFER if defer else 0))
        r = _abi.IterationResult()
        check(lib().vattn_iteration_step(self._h, buf, self._n, flags, -1 if eager_k is None else int(eager_k),
                                         C.byref(r)))
        return IterationResult(bool(r.ok), bool(r.deferred), r.sync_us, r.eager_us, r.reclaim_us,
                               r.reclaimed_groups, r.bg_wait_us, r.sync_bg_wall_us, r.wall_us)

    def bg_wait(self) -> BackgroundResult:
        r = _abi.BgResult()
        check(lib().vattn_bg_wait(self._h, C.byref(r)))
        return BackgroundResult(r.plan_us, r.eager_us, r.reclaim_us, r.reclaimed_groups,
                                r.bg_wall_us, r.waited_us)

    def mark_use(self, stream=None) -> None:
        """Fence for unmaps: work queued on `stream` (default: the current stream of the
        manager's device) so far may read the cache."""
        check(lib().vattn_mark_use(self._h, C.c_void_p(_stream_ptr(stream, self.device))))

    def check_errors(self) -> None:
        """Raise ValueError if a kernel on this cache was asked for rows its slot does not back
        (it clamped them instead of faulting; see vattn_check_errors).  Synchronizes nothing:
        call torch.cuda.synchronize() first to cover every launched kernel."""
        check(lib().vattn_check_errors(self._h))

    # -- parity introspection ---------------------------------------------------------------
    def drain_events(self) -> list[list[int]]:
        n = C.c_int64()
        check(lib().vattn_events(self._h, None, 0, C.byref(n)))
        raw = (C.c_int64 * max(1, 3 * n.value))()
        check(lib().vattn_events(self._h, raw, n.value, C.byref(n)))
        return [[raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]] for i in range(n.value)]

    def parity_state(self) -> dict:
        c = self._counters()
        raw = (C.c_int64 * (5 * self._n))()
        check(lib().vattn_slot_state(self._h, raw, self._n))
        return {
            "slots": [[raw[5 * r], raw[5 * r + 1], raw[5 * r + 2], _PHASES[raw[5 * r + 3]].value,
                       raw[5 * r + 4]] for r in range(self._n)],
            "eager_slot": None if c.eager_slot < 0 else c.eager_slot,
            "created": c.created,
            "mapped": c.mapped,
            "precreated": c.precreated,
            "calls": dict(sorted(self.vmm.calls.items())),
            "total_mapped_bytes": c.total_mapped_bytes,
            "charged_us": c.charged_us,
        }

    def peek_counters(self) -> _abi.Counters:
        """Counters without joining the background thread (monitoring only)."""
        c = _abi.Counters()
        check(lib().vattn_counters_peek(self._h, C.byref(c)))
        return c

    def driver_stats(self, peek: bool = False) -> dict:
        """Measured real-driver cost (CUDA backend)."""
        c = self.peek_counters() if peek else self._counters()
        return {k: getattr(c, k) for k, _ in _abi.Counters._fields_
                if k.startswith(("real_", "init_wall", "spec_", "lazy_"))}

    # -- admission-aware prefetch (B200 addition; logical state untouched) ------------------------
    def predict_alloc(self, k: int) -> list[int]:
        """The next k slots consecutive alloc_reqid() calls would return now."""
        out = (C.c_int32 * max(1, k))()
        n = C.c_int32()
        check(lib().vattn_predict_alloc(self._h, int(k), out, C.byref(n)))
        return list(out[:n.value])

    def prefetch_hint(self, slots, tokens) -> None:
        """Back rows [0, tokens[i]) of slots[i] physically ahead of admission (queued prompts);
        replaces the previous hints; picked up by the next bg_submit(prefetch=True)."""
        n = len(slots)
        sa = (C.c_int32 * max(1, n))(*[int(x) for x in slots])
        ta = (C.c_int64 * max(1, n))(*[int(x) for x in tokens])
        check(lib().vattn_prefetch_hint(self._h, sa, ta, n))

    def foreground(self, active: bool) -> None:
        """Mark the caller's kernel-launch window: the prefetch worker makes no driver call while
        it is active (its cuMemSetAccess calls would otherwise stall the launches)."""
        check(lib().vattn_set_foreground(self._h, int(bool(active))))

    def slot_ready(self, slot: int, tokens: int) -> bool:
        """True when a step growing `slot` to `tokens` rows needs no driver call."""
        r = C.c_int32()
        check(lib().vattn_slot_ready(self._h, int(slot), int(tokens), C.byref(r)))
        return bool(r.value)

    # -- virtual tensors (Table 3 `init` returns the KV cache tensors) ---------
    def _view(self, layer: int, kind: int):
        key = (layer, kind)
        if key in self._views:
            return self._views[key]
        import torch
        g = self._g
        if not 0 <= layer < g.n_layers:
            raise ValueError("layer out of range")
        if g.bytes_per_elem != 2:
            raise ValueError(f"cache views are bfloat16; this geometry has {g.bytes_per_elem}-byte elements")
        row = g.kv_heads_per_worker * g.head_dim          # elements per token row, one layer
        if self.config.sliced:
            # layer l starts l rows into each token's N-layer record: the storage starts there too
            # and ends with the reserved range
            base = self.buffers[kind].device_ptr + layer * row * 2
            token_stride = g.n_layers * row
            size_bytes = self.buffers[0].size - layer * row * 2
        else:
            base = self.buffers[2 * layer + kind].device_ptr
            token_stride = row
            size_bytes = self.buffers[0].size
        dev = torch.device("cuda", self.device)
        storage = torch._C._construct_storage_from_data_pointer(base, dev, size_bytes)
        t = torch.empty(0, dtype=torch.bfloat16, device=dev)
        t.set_(storage, 0, (g.max_batch, g.max_context, g.kv_heads_per_worker, g.head_dim),
               (self.slot_stride // 2, token_stride, g.head_dim, 1))
        self._views[key] = t
        return t

    def k_cache(self, layer: int):
        """[max_batch, max_context, Hkv, D] bf16 view of layer `layer`'s K virtual tensor.
        Only rows backed by step() may be touched."""
        return self._view(layer, 0)

    def v_cache(self, layer: int):
        return self._view(layer, 1)

    def kv_caches(self):
        return [(self.k_cache(i), self.v_cache(i)) for i in range(self._g.n_layers)]


def _stream_ptr(stream, device: int | None = None) -> int:
    if stream is None:
        import torch
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice() if device is None else device)
    return getattr(stream, "cuda_stream", stream) or 0
