"""The C++ allocator core behind the C ABI reproduces the reference bit for bit (CPU, shadow
backend): every recorded reference call script, return values, map/unmap event order, slot
tuples, pool counters, per-API call counts and modelled microseconds."""

import pytest

from allocator_replay import CoreAdapter, load_fixtures, replay

FIXTURES = load_fixtures()


@pytest.mark.parametrize("fixture", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_core_matches_reference_recording(fixture):
    a = CoreAdapter(fixture, backend="shadow")
    try:
        replay(fixture, a)
    finally:
        a.close()
