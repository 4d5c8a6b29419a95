"""pytest plugin: swap the reference KVCacheManager for this package's C-ABI-backed one
before the reference's own test modules are imported (used by test_reference_dropin.py)."""

import os
import sys

REPO = os.environ["VATTN_REPO"]
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ["VATTN_REF"])


def pytest_configure(config):
    import kvsim.manager as ref_manager
    from paper_2405_04437_b200.manager import KVCacheManager

    class DropIn(KVCacheManager):
        def __init__(self, geometry, config):
            super().__init__(geometry, config, backend="shadow", log_events=False)

    import kvsim.vmm as ref_vmm
    from paper_2405_04437_b200 import errors
    errors.use_exception_classes(
        BatchFullError=ref_manager.BatchFullError, DoubleFreeError=ref_manager.DoubleFreeError,
        PoolExhaustedError=ref_vmm.PoolExhaustedError, MappingError=ref_vmm.MappingError,
        AlignmentError=ref_vmm.AlignmentError, InvalidFreeError=ref_vmm.InvalidFreeError,
        LatencyConfigError=ref_vmm.LatencyConfigError)
    ref_manager.KVCacheManager = DropIn
    import kvsim.simulator as ref_sim
    ref_sim.KVCacheManager = DropIn
    import kvsim
    kvsim.KVCacheManager = DropIn
