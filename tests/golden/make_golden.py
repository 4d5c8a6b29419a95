"""Generate allocator golden fixtures by running the REFERENCE itself.

Run in the build container (it imports `kvsim` from /root/reference/pkg/src):

    python tests/golden/make_golden.py

Each fixture is a call script plus, per call, the reference's return value, the ordered
driver events it issued (map/unmap with buffer id and byte offset, captured by wrapping
`VmmDevice.map` / `VmmDevice.unmap_release`, vmm.py:255-297), and the resulting state
(slot tuples, eager slot, pool counters, per-API call counts, modelled µs).  Large scripts
store a SHA-1 digest of the per-call state/events instead of the full objects.

Scripts come from three sources:
  * the reference unit-test scenarios (pkg/tests/test_manager.py),
  * seeded random op streams over several geometries / page-group sizes / pool pressures,
  * the reference serving simulator (kvsim/simulator.py:run) with the manager wrapped in a
    recorder, which captures the exact Algorithm-1 call order (admit → background → step →
    plan → retire) including stale plans.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys
from pathlib import Path

REF = os.environ.get("VATTN_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import kvsim.simulator as ksim  # noqa: E402
from kvsim.geometry import ModelGeometry  # noqa: E402
from kvsim.manager import KVCacheManager, ManagerConfig  # noqa: E402
from kvsim.trace import SimTrace, generate_trace  # noqa: E402
from kvsim.vmm import VmmDevice  # noqa: E402

OUT = Path(__file__).resolve().parent
CHAIN_EVERY = 50
KB64, KB128, KB256, MB2 = 65536, 131072, 262144, 2 * 1024 * 1024
MIB, GIB = 1024 ** 2, 1024 ** 3

# ---------------------------------------------------------------- event capture
_EVENTS: list = []
_orig_map, _orig_unmap = VmmDevice.map, VmmDevice.unmap_release


def _map(self, buffer, offset, handle):
    us = _orig_map(self, buffer, offset, handle)
    _EVENTS.append(("map", buffer.buffer_id, offset))
    return us


def _unmap(self, buffer, offset):
    us = _orig_unmap(self, buffer, offset)
    _EVENTS.append(("unmap", buffer.buffer_id, offset))
    return us


VmmDevice.map, VmmDevice.unmap_release = _map, _unmap


def ref_state(mgr: KVCacheManager) -> dict:
    """Same schema as oracle.allocator.OracleManager.state()."""
    return {
        "slots": [[int(s.active), s.context_len, s.mapped_groups, s.phase.value, s.freed_seq]
                  for s in mgr.slots],
        "eager_slot": mgr.eager_slot,
        "created": mgr.vmm.pool.created,
        "mapped": mgr.vmm.pool.mapped,
        "precreated": mgr.vmm.precreated_available,
        "calls": dict(sorted(mgr.vmm.calls.items())),
        "total_mapped_bytes": mgr.vmm.total_mapped_bytes,
        "charged_us": mgr.vmm.total_charged_us(),
    }


def digest(obj) -> str:
    return hashlib.sha1(json.dumps(obj, sort_keys=True).encode()).hexdigest()


class Recorder:
    """Drives a reference manager from a script, or wraps one driven by the simulator."""

    def __init__(self, mgr: KVCacheManager, full: bool):
        self.mgr, self.full, self.ops = mgr, full, []
        self._plans: dict[int, int] = {}   # id(plan list) -> op index that produced it
        self._chain = ""                   # rolling digest over (events, state) of every call

    def _record(self, entry: dict, ret):
        entry["ret"] = ret
        ev = [[0 if k == "map" else 1, b, o] for k, b, o in _EVENTS]
        st = ref_state(self.mgr)
        if self.full:
            entry["ev"], entry["st"] = ev, st
        else:
            # digest chain; checkpoint every CHAIN_EVERY calls (and the caller adds the last)
            self._chain = digest([self._chain, ev, st])
            if len(self.ops) % CHAIN_EVERY == 0:
                entry["chain"] = self._chain
        _EVENTS.clear()
        self.ops.append(entry)

    def call(self, op: str, **kw):
        _EVENTS.clear()
        m = self.mgr
        try:
            if op == "alloc":
                ret = m.alloc_reqid()
            elif op == "free":
                ret = m.free_reqid(kw["req"])
            elif op == "step":
                r = m.step(list(kw["seq"]))
                ret = [r.ok, r.sync_us]
            elif op == "plan":
                plan = m.plan_overlap(list(kw["seq"]))
                self._plans[id(plan)] = len(self.ops)
                self._last_plan = plan
                ret = [list(p) for p in plan] if self.full else [len(plan), digest([list(p) for p in plan])]
            elif op == "execute":
                plan = kw.pop("_plan_obj")
                src = self._plans.get(id(plan))
                if src is not None:
                    kw["plan_from"] = src
                else:
                    kw["plan"] = [list(p) for p in plan]
                ret = m.execute_plan(plan)
            elif op == "eager":
                ret = m.eager_prepare(kw.get("k"))
            elif op == "reclaim":
                ret = list(m.reclaim())
            elif op == "reclaim_until":
                ret = list(m._reclaim_until(kw["target"]))
            else:
                raise KeyError(op)
        except Exception as exc:  # reference exception -> its class name
            ret = {"error": type(exc).__name__}
        self._record({"op": op, **kw}, ret)
        return ret


def make_fixture(name, geometry: dict, config: dict, script_fn, full=True):
    g = ModelGeometry(**geometry)
    _EVENTS.clear()
    mgr = KVCacheManager(g, ManagerConfig(**config))
    rec = Recorder(mgr, full)
    init = {
        "buffer_count": mgr.buffer_count,
        "groups_per_slot": mgr.groups_per_slot,
        "slot_stride": mgr.slot_stride,
        "buffer_size": mgr.buffers[0].size,
        "init_us": mgr.init_us,
        "state": ref_state(mgr),
    }
    _EVENTS.clear()
    script_fn(rec)
    if not full and rec.ops:
        rec.ops[-1]["chain"] = rec._chain
    return {"name": name, "geometry": geometry, "config": config, "init": init,
            "full": full, "ops": rec.ops}


# ---------------------------------------------------------------- script sources
SMALL = dict(n_layers=3, kv_heads_total=4, head_dim=128, bytes_per_elem=2,
             max_context=4096, max_batch=4)
TINY = dict(n_layers=1, kv_heads_total=2, head_dim=64, bytes_per_elem=2,
            max_context=512, max_batch=2)


def vec(n, lens):
    v = [0] * n
    for r, s in lens.items():
        v[r] = s
    return v


def unit_scripts():
    """Scenarios of pkg/tests/test_manager.py, replayed as scripts."""
    out = []

    def reuse(r):  # test_manager.py:82-89
        for _ in range(4):
            r.call("alloc")
        r.call("step", seq=vec(4, {0: 10, 1: 10, 2: 10, 3: 320}))
        for i in range(4):
            r.call("free", req=i)
        r.call("alloc")
        r.call("free", req=3)
        r.call("free", req=3)            # DoubleFreeError
    out.append(("unit_reuse", SMALL, dict(page_group_size=KB64, pool_bytes=64 * MIB), reuse))

    def batch_full(r):  # :91-96
        for _ in range(5):
            r.call("alloc")
        r.call("step", seq=[5, 0, 0, 0])
        r.call("step", seq=[5000, 0, 0, 0])  # ValueError (length)
    out.append(("unit_batch_full", SMALL, dict(page_group_size=KB64, pool_bytes=64 * MIB), batch_full))

    def failure(r):  # :179-200
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 100}))
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 100, 1: 10}))
        r.call("free", req=0)
        r.call("step", seq=vec(4, {1: 10}))
        r.call("free", req=1)
        r.call("alloc")
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 100, 1: 64}))
    out.append(("unit_failure", SMALL, dict(page_group_size=KB64, pool_bytes=12 * KB64), failure))

    def trim(r):  # :204-213
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 320}))
        r.call("free", req=0)
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 70}))
        for n in (71, 80, 129, 200):
            r.call("step", seq=vec(4, {0: n}))
    out.append(("unit_trim", SMALL, dict(page_group_size=KB64, pool_bytes=64 * MIB), trim))

    def overlap(r):  # :225-273
        r.call("alloc")
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 64, 1: 128}))
        r.call("plan", seq=vec(4, {0: 65, 1: 129}))
        r.call("execute", _plan_obj=r._last_plan)
        r.call("step", seq=vec(4, {0: 65, 1: 129}))
        seq = 60
        for _ in range(10):
            r.call("plan", seq=vec(4, {0: seq + 1, 1: 130}))
            r.call("execute", _plan_obj=r._last_plan)
            seq += 1
            r.call("step", seq=vec(4, {0: seq, 1: 130}))
    out.append(("unit_overlap", SMALL, dict(page_group_size=KB64, pool_bytes=64 * MIB), overlap))

    def eager(r):  # :277-303
        r.call("eager", k=2)
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 192}))
        r.call("eager", k=1)
        r.call("eager", k=1)
        r.call("eager")
        for _ in range(3):
            r.call("alloc")
        r.call("eager", k=1)
    out.append(("unit_eager", SMALL, dict(page_group_size=KB64, pool_bytes=64 * MIB), eager))

    def eager_floor(r):
        r.call("eager", k=2)
        r.call("eager", k=3)
    out.append(("unit_eager_floor", SMALL,
                dict(page_group_size=KB64, pool_bytes=12 * KB64, reclaim_threshold=0.5), eager_floor))

    def reclaim(r):  # :306-342
        r.call("alloc")
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 64, 1: 64}))
        r.call("free", req=0)
        r.call("free", req=1)
        r.call("reclaim")
        r.call("reclaim_until", target=24 * KB64 - 6 * KB64)
        r.call("reclaim_until", target=24 * KB64)
    out.append(("unit_reclaim_order", SMALL,
                dict(page_group_size=KB64, pool_bytes=24 * KB64, reclaim_threshold=0.0), reclaim))

    def reclaim_thr(r):
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 128}))
        r.call("reclaim")
        r.call("free", req=0)
        r.call("reclaim")
    out.append(("unit_reclaim_threshold", SMALL,
                dict(page_group_size=KB64, pool_bytes=12 * KB64, reclaim_threshold=0.5), reclaim_thr))

    def precreate_half(r):  # :69-72 then re-creation after release (Appendix A.4)
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 300}))
        r.call("free", req=0)
        r.call("reclaim_until", target=32 * KB64)
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 400}))
    out.append(("unit_precreate_half", SMALL,
                dict(page_group_size=KB64, pool_bytes=32 * KB64, pre_create_fraction=0.5),
                precreate_half))

    def y34(r):  # :152-159
        r.call("alloc")
        r.call("step", seq=vec(4, {0: 2048}))
        r.call("step", seq=vec(4, {0: 2049}))
    y34g = dict(n_layers=60, kv_heads_total=8, head_dim=128, bytes_per_elem=2,
                max_context=200_000, max_batch=4, tp_degree=2)
    out.append(("unit_yi34b_tp2_crossing", y34g, dict(page_group_size=MB2, pool_bytes=4 * GIB), y34))

    def tiny(r):  # BASELINE config 1
        r.call("alloc")
        r.call("alloc")
        r.call("step", seq=[128, 512])
        r.call("plan", seq=[129, 512])
        r.call("free", req=1)
        r.call("alloc")
        r.call("step", seq=[129, 300])
        r.call("free", req=0)
        r.call("free", req=1)
        r.call("reclaim_until", target=64 * MIB)
    out.append(("config1_tiny", TINY, dict(page_group_size=MB2, pool_bytes=64 * MIB), tiny))
    return out


def random_script(seed, n_ops, max_batch, max_context, group_cap=None):
    def fn(r):
        rng = random.Random(seed)
        seq = [0] * max_batch
        active: set[int] = set()
        plan = []
        for _ in range(n_ops):
            x = rng.random()
            if x < 0.18:
                ret = r.call("alloc")
                if isinstance(ret, int):
                    active.add(ret)
                    seq[ret] = rng.randint(0, max_context)
            elif x < 0.30 and active:
                rid = rng.choice(sorted(active))
                active.discard(rid)
                seq[rid] = 0
                r.call("free", req=rid)
            elif x < 0.33:
                r.call("free", req=rng.randrange(max_batch))   # may be DoubleFreeError
            elif x < 0.43:
                nxt = [min(s + rng.randint(0, 3), max_context) if i in active else 0
                       for i, s in enumerate(seq)]
                r.call("plan", seq=nxt)
                plan = r._last_plan
            elif x < 0.50:
                r.call("execute", _plan_obj=plan)
            elif x < 0.56:
                r.call("eager", k=rng.choice([None, 0, 1, 2, 3, 50]))
            elif x < 0.61:
                r.call("reclaim")
            elif x < 0.63:
                r.call("step", seq=[max_context + 1] + [0] * (max_batch - 1))  # ValueError
            else:
                for i in active:
                    seq[i] = min(seq[i] + rng.choice([0, 1, 1, 1, 7, 64]), max_context)
                ret = r.call("step", seq=list(seq))
                if isinstance(ret, list) and not ret[0]:
                    # serving-layer preemption of the newest active slot
                    rid = max(active)
                    active.discard(rid)
                    seq[rid] = 0
                    r.call("free", req=rid)
    return fn


def random_fixtures():
    out = []
    cases = [
        ("rand_small_64k", SMALL | dict(max_batch=6), dict(page_group_size=KB64, pool_bytes=40 * MIB), 4096),
        ("rand_small_64k_tight", SMALL | dict(max_batch=6), dict(page_group_size=KB64, pool_bytes=30 * KB64,
                                                                  reclaim_threshold=0.2, pre_create_fraction=0.5), 700),
        ("rand_small_128k_eager", SMALL | dict(max_batch=5), dict(page_group_size=KB128, pool_bytes=12 * MIB,
                                                                   eager_groups=2, reclaim_threshold=0.3), 3000),
        ("rand_small_256k", SMALL | dict(max_batch=5), dict(page_group_size=KB256, pool_bytes=48 * KB256,
                                                             pre_create_fraction=0.25), 4096),
        ("rand_small_2m", SMALL | dict(max_batch=6), dict(page_group_size=MB2, pool_bytes=96 * MB2,
                                                           reclaim_threshold=0.25), 4096),
        ("rand_sliced_2m", SMALL | dict(max_batch=6), dict(page_group_size=MB2, pool_bytes=40 * MB2,
                                                            sliced=True, eager_groups=1), 4096),
        ("rand_sliced_64k", SMALL | dict(max_batch=4), dict(page_group_size=KB64, pool_bytes=60 * KB64,
                                                             sliced=True), 2000),
        ("rand_tiny_2m", TINY, dict(page_group_size=MB2, pool_bytes=3 * MB2), 512),
        ("rand_l8_2m_tight", dict(n_layers=4, kv_heads_total=8, head_dim=128, bytes_per_elem=2,
                                  max_context=8192, max_batch=8),
         dict(page_group_size=MB2, pool_bytes=60 * MB2, eager_groups=2, reclaim_threshold=0.1), 8192),
    ]
    for i, (name, g, cfg, ctx) in enumerate(cases):
        for rep in range(2):
            seed = 1000 * i + rep
            out.append((f"{name}_s{seed}", g, cfg, random_script(seed, 400, g["max_batch"], min(ctx, g["max_context"]))))
    return out


# ---------------------------------------------------------------- simulator capture
def simulator_fixture(name, trace, geometry: dict, full=False, **run_kw):
    """Record the reference simulator's exact manager call sequence."""
    holder = {}
    pg, pool = run_kw["page_group_size"], run_kw["pool_bytes"]
    cfg = dict(page_group_size=int(pg), pool_bytes=pool,
               reclaim_threshold=run_kw.get("reclaim_threshold", 0.10),
               eager_groups=run_kw.get("eager_groups", 0),
               sliced=run_kw.get("sliced", False),
               pre_create_fraction=run_kw.get("pre_create_fraction", 1.0))

    class Wrapped:
        def __init__(self, g, config):
            _EVENTS.clear()
            self._m = KVCacheManager(g, config)
            self._rec = Recorder(self._m, full)
            holder["rec"] = self._rec
            holder["init"] = {
                "buffer_count": self._m.buffer_count, "groups_per_slot": self._m.groups_per_slot,
                "slot_stride": self._m.slot_stride, "buffer_size": self._m.buffers[0].size,
                "init_us": self._m.init_us, "state": ref_state(self._m),
            }
            self.init_us = self._m.init_us
            self.vmm = self._m.vmm
            _EVENTS.clear()

        def __getattr__(self, k):
            return getattr(self._m, k)

        def alloc_reqid(self):
            ret = self._rec.call("alloc")
            if isinstance(ret, dict):
                from kvsim.manager import BatchFullError
                raise BatchFullError("full")
            return ret

        def free_reqid(self, rid):
            self._rec.call("free", req=rid)

        def step(self, seq):
            ok, us = self._rec.call("step", seq=list(seq))
            from kvsim.manager import StepResult
            return StepResult(ok=ok, sync_us=us)

        def plan_overlap(self, seq):
            self._rec.call("plan", seq=list(seq))
            return self._rec._last_plan

        def execute_plan(self, plan):
            return self._rec.call("execute", _plan_obj=plan)

        def eager_prepare(self, k=None):
            return self._rec.call("eager", k=k) if k is not None else self._rec.call("eager")

        def reclaim(self):
            return tuple(self._rec.call("reclaim"))

    saved = ksim.KVCacheManager
    ksim.KVCacheManager = Wrapped
    try:
        metrics = ksim.run(trace, ModelGeometry(**geometry), **run_kw)
    finally:
        ksim.KVCacheManager = saved
    rec = holder["rec"]
    rec.ops[-1]["chain"] = rec._chain
    summary = metrics.summary()
    return {"name": name, "geometry": geometry, "config": cfg, "init": holder["init"],
            "full": full, "ops": rec.ops,
            "sim": {"iterations": summary["iterations"], "stall_ms_total": summary["stall_ms_total"],
                    "preemptions": summary["preemptions"]}}


def simulator_fixtures():
    out = []
    y34 = dict(n_layers=60, kv_heads_total=8, head_dim=128, bytes_per_elem=2,
               max_context=200_000, max_batch=8, tp_degree=2)
    spike = SimTrace.from_rows([(0, p, 8) for p in (2047, 2047, 6142, 2045, 2047)])
    for mode in ("sync", "overlapped"):   # test_acceptance.py:113-142
        out.append(simulator_fixture(f"sim_spike_{mode}", spike, y34, full=False,
                                     page_group_size=MB2, mode=mode, pool_bytes=8 * GIB))
    small = dict(n_layers=3, kv_heads_total=4, head_dim=128, bytes_per_elem=2,
                 max_context=4096, max_batch=3)
    shapes = [(1, 1), (63, 3), (65, 3), (126, 30)]   # test_acceptance.py:256
    k = 0
    for combo in [(0, 1, 2), (3, 3, 1), (2, 0, 3, 1), (1, 1, 1, 1, 1), (3, 2, 1, 0, 3)]:
        trace = SimTrace.from_rows([(0, *shapes[c]) for c in combo])
        for mode in ("sync", "overlapped"):
            for eager in (0, 2):
                for thr in (0.1, 0.9):
                    out.append(simulator_fixture(
                        f"sim_grid{k}_{mode}_e{eager}_t{thr}", trace, small, full=True,
                        page_group_size=KB64, mode=mode, eager_groups=eager,
                        reclaim_threshold=thr, pool_bytes=16 * MIB))
        k += 1
    # preemption under a tiny pool (test_simulator.py:135-154)
    pre = SimTrace.from_rows([(0, 64, 10), (0, 64, 4)])
    for mode in ("sync", "overlapped"):
        out.append(simulator_fixture(f"sim_preempt_{mode}", pre, dict(small, max_batch=8), full=True,
                                     page_group_size=KB64, mode=mode, pool_bytes=12 * KB64,
                                     preemption_cap=100_000))
    # config 5 at Llama-3-8B shape (2 MiB, eager auto, reclaim 0.10), reduced request count
    l8 = dict(n_layers=32, kv_heads_total=8, head_dim=128, bytes_per_elem=2,
              max_context=4096, max_batch=64)
    trace = generate_trace(96, qps=16.0, prompt_dist="uniform:128:3072",
                           decode_dist="uniform:16:256", seed=0, max_total_tokens=4096)
    eager = ksim.median_prompt_groups(trace, ModelGeometry(**l8), MB2)
    for mode in ("sync", "overlapped"):
        out.append(simulator_fixture(f"sim_config5_l8_{mode}", trace, l8, full=False,
                                     page_group_size=MB2, mode=mode, pool_bytes=6 * GIB,
                                     eager_groups=eager, reclaim_threshold=0.10,
                                     preemption_cap=100_000))
    return out


def main():
    fixtures = []
    for name, g, cfg, fn in unit_scripts():
        fixtures.append(make_fixture(name, g, cfg, fn, full=True))
    for name, g, cfg, fn in random_fixtures():
        fixtures.append(make_fixture(name, g, cfg, fn, full=True))
    fixtures.extend(simulator_fixtures())
    path = OUT / "allocator_golden.json.gz"
    with gzip.open(path, "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": REF,
                   "fixtures": fixtures}, fh, separators=(",", ":"))
    n_ops = sum(len(f["ops"]) for f in fixtures)
    print(f"wrote {path} ({path.stat().st_size} B): {len(fixtures)} fixtures, {n_ops} calls")


if __name__ == "__main__":
    main()
