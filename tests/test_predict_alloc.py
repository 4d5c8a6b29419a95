"""predict_alloc (admission-aware prefetch) names exactly the slots the next alloc_reqid calls
return, on the shadow backend over random op streams (eager slot first, then the reference's
(mapped_groups, -req_id) ranking, manager.py:163-178)."""

import random

import pytest

MB = 1 << 20


@pytest.mark.parametrize("seed", range(6))
def test_predict_alloc_matches_alloc_reqid(seed):
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.errors import BatchFullError

    rng = random.Random(seed)
    g = ModelGeometry(2, 2, 64, 2, max_context=8192, max_batch=6)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=64 * 1024, pool_bytes=256 * MB,
                                          eager_groups=rng.choice([0, 1, 3]), reclaim_threshold=0.1),
                         backend="shadow")
    lens = [0] * 6
    for _ in range(120):
        op = rng.random()
        if op < 0.3:
            k = rng.randint(1, 6)
            pred = mgr.predict_alloc(k)
            got = []
            try:
                for _ in range(len(pred)):
                    got.append(mgr.alloc_reqid())
            except BatchFullError:
                pass
            assert got == pred
            for r in got:
                lens[r] = rng.randint(1, 3000)
            if len(pred) < k:
                with pytest.raises(BatchFullError):
                    mgr.alloc_reqid()
        elif op < 0.5:
            act = [r for r in range(6) if lens[r]]
            if act:
                r = rng.choice(act)
                mgr.free_reqid(r)
                lens[r] = 0
        elif op < 0.6:
            mgr.eager_prepare()
        else:
            lens = [min(x + rng.choice([1, 50, 700]), 8192) if x else 0 for x in lens]
            if not mgr.step(lens).ok:
                for r in range(6):
                    if lens[r]:
                        mgr.free_reqid(r)
                        lens[r] = 0
                        break
        # readiness on the shadow backend == logically mapped prefix
        for r in range(6):
            n = mgr.slots[r].mapped_groups * (64 * 1024) // mgr.per_buffer_token_bytes
            assert mgr.slot_ready(r, n)
            if mgr.slots[r].mapped_groups < mgr.groups_per_slot:
                assert not mgr.slot_ready(r, n + 1)
    mgr.close()
