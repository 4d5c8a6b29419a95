"""Exception classes with the reference's names and bases (manager.py:28-33, vmm.py:26-47).

The reference is imported nowhere; a caller catching `BatchFullError` or `PoolExhaustedError`
by name keeps working after swapping in this package.
"""


class BatchFullError(RuntimeError):
    """All request slots are active (manager.py:28)."""


class DoubleFreeError(RuntimeError):
    """free_reqid on an inactive slot (manager.py:32)."""


class VmmError(Exception):
    """Base of virtual-memory management failures (vmm.py:26)."""


class AlignmentError(VmmError):
    pass


class PoolExhaustedError(VmmError):
    pass


class MappingError(VmmError):
    pass


class InvalidFreeError(VmmError):
    pass


class LatencyConfigError(VmmError):
    pass


class CudaError(RuntimeError):
    """A CUDA driver/runtime call failed inside libvattn."""


class UnsupportedError(ValueError):
    """Shape or layout not covered by the sm_100a kernels."""


class NativeLibraryMissing(RuntimeError):
    """libvattn.so is not built; there is no Python fallback by design."""


_BY_STATUS = {
    1: BatchFullError,
    2: DoubleFreeError,
    3: ValueError,
    4: PoolExhaustedError,
    5: MappingError,
    6: AlignmentError,
    7: InvalidFreeError,
    8: LatencyConfigError,
    9: CudaError,
    10: UnsupportedError,
    11: RuntimeError,
}


def from_status(status: int, msg: str) -> Exception:
    return _BY_STATUS.get(status, RuntimeError)(msg)


def use_exception_classes(**classes) -> None:
    """Raise the caller's own exception classes instead of ours, e.g. when swapping this
    package in under code that catches `kvsim.manager.BatchFullError`:

        use_exception_classes(BatchFullError=kvsim.manager.BatchFullError, ...)
    """
    names = {v.__name__: k for k, v in _BY_STATUS.items()}
    for name, cls in classes.items():
        if name not in names:
            raise KeyError(f"unknown exception name {name!r}")
        _BY_STATUS[names[name]] = cls
        globals()[name] = cls
