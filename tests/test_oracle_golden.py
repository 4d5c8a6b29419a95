"""Pin the CPU oracle to the reference: replay every recorded reference call script."""

import pytest

from allocator_replay import OracleAdapter, load_fixtures, replay

FIXTURES = load_fixtures()


@pytest.mark.parametrize("fixture", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_oracle_matches_reference_recording(fixture):
    replay(fixture, OracleAdapter(fixture))


def test_fixture_coverage():
    """The golden set exercises every reference behaviour the survey lists (Appendix A)."""
    ops = {}
    errors = set()
    unmaps = 0
    for f in FIXTURES:
        for e in f["ops"]:
            ops[e["op"]] = ops.get(e["op"], 0) + 1
            if isinstance(e["ret"], dict):
                errors.add(e["ret"]["error"])
            if f["full"]:
                unmaps += sum(1 for ev in e["ev"] if ev[0] == 1)
    assert set(ops) == {"alloc", "free", "step", "plan", "execute", "eager", "reclaim", "reclaim_until"}
    assert {"BatchFullError", "DoubleFreeError", "ValueError"} <= errors
    assert unmaps > 100
    failed_steps = sum(1 for f in FIXTURES for e in f["ops"]
                       if e["op"] == "step" and isinstance(e["ret"], list) and not e["ret"][0])
    assert failed_steps > 5
