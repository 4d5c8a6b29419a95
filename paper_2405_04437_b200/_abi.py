"""ctypes binding of include/vattn.h (libvattn.so, built in-tree by build.py).

This is the Python side of the C-ABI boundary: plain pointers, ints and structs only.
Status codes are mapped 1:1 onto the reference exception classes (errors.py).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvattn.so"

c_i32, c_i64, c_u32, c_u64, c_f32, c_f64, c_vp = (C.c_int32, C.c_int64, C.c_uint32, C.c_uint64,
                                                  C.c_float, C.c_double, C.c_void_p)
P_i64 = C.POINTER(c_i64)
P_i32 = C.POINTER(c_i32)
P_f64 = C.POINTER(c_f64)


class LatencyEntry(C.Structure):
    _fields_ = [("api", C.c_char_p), ("page_group_bytes", c_i64), ("us", c_f64)]


class Config(C.Structure):
    _fields_ = [
        ("n_layers", c_i32), ("kv_heads_total", c_i32), ("head_dim", c_i32),
        ("bytes_per_elem", c_i32), ("tp_degree", c_i32), ("n_q_heads_total", c_i32),
        ("max_context", c_i64), ("max_batch", c_i64),
        ("page_group_size", c_i64), ("pool_bytes", c_i64),
        ("reclaim_threshold", c_f64), ("pre_create_fraction", c_f64),
        ("eager_groups", c_i64), ("sliced", c_i32),
        ("backend", c_i32), ("device", c_i32), ("release_physical", c_i32),
        ("log_events", c_i32), ("batch_set_access", c_i32),
        ("latency", C.POINTER(LatencyEntry)), ("n_latency", c_i32), ("prefetch_tokens", c_i32),
        ("prefetch_slots", c_i32), ("prefetch_slot_tokens", c_i32), ("lazy_unmap", c_i32),
        ("phys_chunk_groups", c_i32),
    ]


class StepResultC(C.Structure):
    _fields_ = [("ok", c_i32), ("sync_us", c_f64), ("wall_us", c_f64), ("bg_wait_us", c_f64)]


class Counters(C.Structure):
    _fields_ = [(n, c_i64) for n in (
        "created", "mapped", "precreated", "total_mapped_bytes", "capacity", "page_group_size",
        "buffer_count", "groups_per_slot", "slot_stride", "buffer_size",
        "per_buffer_token_bytes", "max_batch", "max_context", "eager_slot", "next_handle_id")] + [
        ("init_us", c_f64), ("charged_us", c_f64)] + [(n, c_i64) for n in (
            "real_maps", "real_unmaps", "real_set_access_calls", "real_creates", "real_releases")] + [
        (n, c_f64) for n in ("real_map_wall_us", "real_unmap_wall_us", "real_create_wall_us",
                             "real_set_access_wall_us", "init_wall_us")] + [
        (n, c_i64) for n in ("spec_maps", "spec_hits", "spec_steals", "spec_pages", "lazy_unmaps",
                             "phys_chunk_groups", "phys_chunks_mapped", "phys_mapped_bytes")]


class BgResult(C.Structure):
    _fields_ = [("plan_us", c_f64), ("eager_us", c_f64), ("reclaim_us", c_f64),
                ("reclaimed_groups", c_i64), ("bg_wall_us", c_f64), ("waited_us", c_f64)]


class CacheDesc(C.Structure):
    _fields_ = [("k_base", c_vp), ("v_base", c_vp), ("slot_stride_bytes", c_i64),
                ("token_stride_bytes", c_i64), ("slot_tokens", c_i32), ("n_slots", c_i32),
                ("n_kv_heads", c_i32), ("head_dim", c_i32)]


class RotaryC(C.Structure):
    _fields_ = [("cos", c_vp), ("sin", c_vp), ("rotary_dim", c_i32), ("interleaved", c_i32)]


class IterationResult(C.Structure):
    _fields_ = [("ok", c_i32), ("deferred", c_i32), ("sync_us", c_f64), ("eager_us", c_f64),
                ("reclaim_us", c_f64), ("reclaimed_groups", c_i64), ("bg_wait_us", c_f64),
                ("sync_bg_wall_us", c_f64), ("wall_us", c_f64)]


BG_EXECUTE_PLAN, BG_EAGER, BG_RECLAIM, BG_CREDIT, ITER_DEFER, BG_PREFETCH = 1, 2, 4, 8, 16, 32

# every symbol include/vattn.h declares, with its ctypes signature
SIGNATURES = {
    "vattn_last_error": (C.c_char_p, []),
    "vattn_abi_version": (c_i32, []),
    "vattn_abi_sizes": (c_i32, [C.POINTER(c_i64), c_i32]),
    "vattn_create": (c_i32, [C.POINTER(Config), C.POINTER(c_vp)]),
    "vattn_destroy": (c_i32, [c_vp]),
    "vattn_alloc_reqid": (c_i32, [c_vp, P_i32]),
    "vattn_free_reqid": (c_i32, [c_vp, c_i32]),
    "vattn_step": (c_i32, [c_vp, P_i64, c_i32, C.POINTER(StepResultC)]),
    "vattn_iteration_step": (c_i32, [c_vp, P_i64, c_i32, c_u32, c_i64, C.POINTER(IterationResult)]),
    "vattn_plan_overlap": (c_i32, [c_vp, P_i64, c_i32, P_i64]),
    "vattn_plan_fetch": (c_i32, [c_vp, P_i64, c_i64]),
    "vattn_execute_plan": (c_i32, [c_vp, P_i64, c_i64, P_f64]),
    "vattn_eager_prepare": (c_i32, [c_vp, c_i64, P_f64]),
    "vattn_reclaim": (c_i32, [c_vp, P_i64, P_f64]),
    "vattn_reclaim_until": (c_i32, [c_vp, c_i64, P_i64, P_f64]),
    "vattn_bg_submit": (c_i32, [c_vp, P_i64, c_i64, c_u32, c_i64]),
    "vattn_bg_wait": (c_i32, [c_vp, C.POINTER(BgResult)]),
    "vattn_mark_use": (c_i32, [c_vp, c_vp]),
    "vattn_check_errors": (c_i32, [c_vp]),
    "vattn_counters_get": (c_i32, [c_vp, C.POINTER(Counters)]),
    "vattn_counters_peek": (c_i32, [c_vp, C.POINTER(Counters)]),
    "vattn_slot_state": (c_i32, [c_vp, P_i64, c_i64]),
    "vattn_api_count": (c_i32, []),
    "vattn_api_name": (C.c_char_p, [c_i32]),
    "vattn_api_stats": (c_i32, [c_vp, P_i64, P_f64, P_i32, P_i32]),
    "vattn_buffer_mappings": (c_i32, [c_vp, c_i32, P_i64, P_i64, c_i64, P_i64]),
    "vattn_events": (c_i32, [c_vp, P_i64, c_i64, P_i64]),
    "vattn_buffer_base": (c_i32, [c_vp, c_i32, C.POINTER(c_u64)]),
    "vattn_predict_alloc": (c_i32, [c_vp, c_i32, P_i32, P_i32]),
    "vattn_set_foreground": (c_i32, [c_vp, c_i32]),
    "vattn_prefetch_hint": (c_i32, [c_vp, P_i32, P_i64, c_i32]),
    "vattn_slot_ready": (c_i32, [c_vp, c_i32, c_i64, P_i32]),
    "vattn_kv_append": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "vattn_decode": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_f32, c_i32, c_vp]),
    "vattn_decode_append": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_f32, c_i32, c_vp]),
    "vattn_decode_append_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                        c_f32, c_i32, c_vp, c_i64, c_vp]),
    "vattn_kv_append_rotary": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, C.POINTER(RotaryC), c_vp]),
    "vattn_kv_append_rotary_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                           C.POINTER(RotaryC), c_vp]),
    "vattn_prefill_varlen": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, P_i32, P_i32, P_i32, P_i32, c_f32, c_i32, c_vp]),
    "vattn_prefill_varlen_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, P_i32, P_i32, P_i32, P_i32,
                                         c_f32, c_i32, c_vp]),
    "vattn_prefill_rotary": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32, c_f32, c_i32,
                                     C.POINTER(RotaryC), c_vp]),
    "vattn_prefill_rotary_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_f32,
                                         c_i32, C.POINTER(RotaryC), c_vp]),
    "vattn_decode_append_rotary": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_f32, c_i32,
                                           C.POINTER(RotaryC), c_vp]),
    "vattn_decode_append_rotary_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                               c_f32, c_i32, C.POINTER(RotaryC), c_vp, c_i64, c_vp]),
    "vattn_prefill": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32, c_f32, c_i32, c_vp]),
    "vattn_kv_append_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "vattn_decode_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_f32,
                                 c_i32, c_vp, c_i64, c_vp]),
    "vattn_prefill_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_i32, c_i32, c_i32, c_i32,
                                  c_f32, c_i32, c_vp]),
    "vattn_decode_paged": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_vp,
                                   c_i32, c_i32, c_vp, c_f32, c_i32, c_vp, c_i64, c_vp]),
    "vattn_kv_append_paged": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_i32,
                                      c_vp, c_vp]),
    "vattn_prefill_paged": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_vp, c_i32, c_i32,
                                    c_f32, c_i32, c_vp]),
    "vattn_vmm_microbench": (c_i32, [c_i32, c_i64, c_i32, c_i32, C.POINTER(c_f64)]),
    "vattn_vmm_slice_probe": (c_i32, [c_i32, c_i32, c_i32, c_i32, C.POINTER(c_f64)]),
    "vattn_vmm_parallel_probe": (c_i32, [c_i32, c_i32, c_i32, C.POINTER(c_f64)]),
    "vattn_compute_proxy": (c_i32, [c_u64, c_vp]),
    "vattn_decode_num_splits": (c_i32, [c_i32, c_i32, c_i32]),
    "vattn_decode_workspace_bytes": (c_i64, [c_i32, c_i32, c_i32, c_i32]),
    "vattn_decode_kernel_name": (c_i32, [c_i32, c_i32, c_i32, c_i32, c_i32, C.c_char_p, c_i32]),
    "vattn_gather_create": (c_i32, [c_i32, c_i32, c_i32, c_i64, C.POINTER(c_vp), c_vp]),
    "vattn_gather_open": (c_i32, [c_vp, c_vp]),
    "vattn_gather_create_local": (c_i32, [c_i32, c_i32, c_i64, C.POINTER(c_vp)]),
    "vattn_gather_output": (c_i32, [c_vp, C.POINTER(c_u64)]),
    "vattn_gather_wait": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "vattn_gather_check": (c_i32, [c_vp, C.POINTER(c_u32)]),
    "vattn_gather_destroy": (c_i32, [c_vp]),
    "vattn_decode_gather": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_f32, c_i32, c_vp]),
    "vattn_decode_gather_raw": (c_i32, [C.POINTER(CacheDesc), c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                        c_f32, c_i32, c_vp, c_i64, c_vp]),
}

IPC_HANDLE_BYTES = 64

_lib = None
_lock = threading.Lock()


def lib():
    """Load libvattn.so.  No fallback: a missing library is an error (the product path is native)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                if os.environ.get("VATTN_NO_AUTOBUILD"):
                    raise errors.NativeLibraryMissing(f"{LIB_PATH} not built")
                from .build import build
                build()
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().vattn_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)


def api_names() -> list[str]:
    L = lib()
    return [L.vattn_api_name(i).decode() for i in range(L.vattn_api_count())]
