"""B200-native vAttention hot path: virtual-memory KV allocator (C++ core over cuMem* at 2 MiB),
background mapping thread, and sm_100a KV-append / decode / prefill attention kernels.

Drop-in for the reference allocator API (kvsim.manager.KVCacheManager); see INTEGRATION.md.
"""

from .errors import (AlignmentError, BatchFullError, DoubleFreeError, InvalidFreeError,  # noqa: F401
                     LatencyConfigError, MappingError, PoolExhaustedError, VmmError)
from .geometry import ModelGeometry, block_size_tokens, prefill_page_groups  # noqa: F401
from .manager import (KVCacheManager, ManagerConfig, Phase, RequestSlot, StepResult)  # noqa: F401

__all__ = [
    "KVCacheManager", "ManagerConfig", "Phase", "RequestSlot", "StepResult", "ModelGeometry",
    "block_size_tokens", "prefill_page_groups", "BatchFullError", "DoubleFreeError", "VmmError",
    "AlignmentError", "PoolExhaustedError", "MappingError", "InvalidFreeError", "LatencyConfigError",
]
