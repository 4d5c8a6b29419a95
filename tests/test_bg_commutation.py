"""The background-thread protocol preserves the reference state exactly.

1. vattn_iteration_step with VATTN_ITER_DEFER (eager_prepare/reclaim queued behind step when
   provably equivalent) reaches the same allocator state as the reference order
   (eager -> reclaim -> step, simulator.py:414-426) at every quiescent point.
2. execute_plan submitted early with plan credits (during the previous iteration) leaves
   alloc_reqid's slot choice identical to the reference order (admit before execute_plan).
"""

import random

import pytest

from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry

KB64, MB2 = 65536, 2 * 1024 * 1024


def _state(m):
    st = m.parity_state()
    return st["slots"], st["eager_slot"], st["created"], st["mapped"], st["calls"], st["total_mapped_bytes"]


@pytest.mark.parametrize("seed", range(12))
def test_deferred_eager_reclaim_equals_reference_order(seed):
    rng = random.Random(seed)
    g = ModelGeometry(3, 4, 128, 2, max_context=4096, max_batch=6)
    pg = [KB64, MB2][seed % 2]
    pool = rng.choice([20, 40, 200]) * (6 * pg)
    cfg = ManagerConfig(page_group_size=pg, pool_bytes=pool, eager_groups=rng.randint(0, 3),
                        reclaim_threshold=rng.choice([0.0, 0.1, 0.3]),
                        pre_create_fraction=rng.choice([0.5, 1.0]))
    a = KVCacheManager(g, cfg, backend="shadow")      # reference order
    b = KVCacheManager(g, cfg, backend="shadow")      # deferred when safe
    seq = [0] * 6
    deferred = 0
    for _ in range(300):
        x = rng.random()
        if x < 0.2:
            try:
                ra = a.alloc_reqid()
            except Exception as e:                     # BatchFull on both
                with pytest.raises(type(e)):
                    b.alloc_reqid()
                continue
            assert b.alloc_reqid() == ra
            seq[ra] = rng.randint(1, 1500)
        elif x < 0.35:
            act = [i for i, s in enumerate(seq) if s]
            if act:
                r = rng.choice(act)
                a.free_reqid(r)
                b.free_reqid(r)
                seq[r] = 0
        else:
            for i, s in enumerate(seq):
                if s:
                    seq[i] = min(4096, s + rng.choice([1, 1, 3, 64]))
            ra = a.iteration_step(seq, defer=False)
            rb = b.iteration_step(seq, defer=True)
            b.bg_wait()
            assert ra.ok == rb.ok
            deferred += rb.deferred
            if not ra.ok:           # preempt the highest active slot on both
                r = max(i for i, s in enumerate(seq) if s)
                a.free_reqid(r)
                b.free_reqid(r)
                seq[r] = 0
            assert _state(a) == _state(b)
    assert deferred > 0


@pytest.mark.parametrize("seed", range(12))
def test_early_plan_with_credits_keeps_admission_choice(seed):
    """Reference: retire -> admit -> execute_plan.  Ours: execute_plan (bg, credits) -> retire -> admit."""
    rng = random.Random(100 + seed)
    g = ModelGeometry(2, 4, 128, 2, max_context=2048, max_batch=5)
    cfg = ManagerConfig(page_group_size=KB64, pool_bytes=400 * KB64)
    a = KVCacheManager(g, cfg, backend="shadow")
    b = KVCacheManager(g, cfg, backend="shadow")
    seq = [0] * 5
    for _ in range(200):
        nxt = [s + 1 if s else 0 for s in seq]
        plan_a = a.plan_overlap(nxt)
        plan_b = b.plan_overlap(nxt)
        assert plan_a == plan_b
        b.bg_submit(plan_b, credit=True)              # ours: runs before retire/admit
        # retire some (both); stale plans then map into freed slots (Appendix A.6)
        for r in [i for i, s in enumerate(seq) if s]:
            if rng.random() < 0.3:
                a.free_reqid(r)
                b.free_reqid(r)
                seq[r] = 0
                nxt[r] = 0
        # admit (both) — b's choice must ignore the groups its early plan added
        for _ in range(rng.randint(0, 2)):
            try:
                ra = a.alloc_reqid()
            except Exception:
                continue
            assert b.alloc_reqid() == ra
            seq[ra] = nxt[ra] = rng.randint(1, 600)
        a.execute_plan(plan_a)                        # reference position
        for i, s in enumerate(seq):
            if s:
                seq[i] = nxt[i]
        assert a.step(seq).ok == b.step(seq).ok
        assert _state(a) == _state(b)
