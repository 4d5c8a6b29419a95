"""Replay the reference-recorded allocator scripts (tests/golden/allocator_golden.json.gz)
through an implementation adapter and compare every call bit for bit.

An adapter exposes:  call(op, **kw) -> ret  (same encoding as make_golden.Recorder),
events() -> [[0|1, buffer_id, offset], ...] since the previous call, state() -> dict,
init_info() -> dict.  Used for the CPU oracle and for the C-ABI allocator core.
"""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "allocator_golden.json.gz"


def load_fixtures():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)["fixtures"]


def digest(obj) -> str:
    return hashlib.sha1(json.dumps(obj, sort_keys=True).encode()).hexdigest()


def _norm_ret(op, ret, full):
    if op == "plan" and not isinstance(ret, dict):
        plan = [list(p) for p in ret]
        return plan if full else [len(plan), digest(plan)]
    if isinstance(ret, tuple):
        return list(ret)
    return ret


def replay(fixture: dict, adapter) -> None:
    """Raise AssertionError with the first diverging call."""
    name = fixture["name"]
    info = adapter.init_info()
    for key in ("buffer_count", "groups_per_slot", "slot_stride", "buffer_size", "init_us"):
        assert info[key] == fixture["init"][key], (name, "init", key, info[key], fixture["init"][key])
    assert adapter.state() == fixture["init"]["state"], (name, "init state")
    adapter.events()
    plans: dict[int, list] = {}
    chain = ""
    full = fixture["full"]
    for i, entry in enumerate(fixture["ops"]):
        op = entry["op"]
        kw = {}
        if op == "free":
            kw["req"] = entry["req"]
        elif op in ("step", "plan"):
            kw["seq"] = entry["seq"]
        elif op == "execute":
            kw["plan"] = plans[entry["plan_from"]] if "plan_from" in entry else entry["plan"]
        elif op == "eager":
            kw["k"] = entry.get("k")
        elif op == "reclaim_until":
            kw["target"] = entry["target"]
        ret = adapter.call(op, **kw)
        if op == "plan" and not isinstance(ret, dict):
            plans[i] = [list(p) for p in ret]
        got = _norm_ret(op, ret, full)
        assert got == entry["ret"], (name, i, op, "ret", got, entry["ret"])
        ev = adapter.events()
        st = adapter.state()
        if full:
            assert ev == entry["ev"], (name, i, op, "events", ev[:8], entry["ev"][:8])
            assert st == entry["st"], (name, i, op, "state", st, entry["st"])
        else:
            chain = digest([chain, ev, st])
            if "chain" in entry:
                assert chain == entry["chain"], (name, i, op, "chain digest")


class OracleAdapter:
    """Adapter over oracle.allocator.OracleManager."""

    def __init__(self, fixture):
        from oracle.allocator import Geometry, OracleError, OracleManager

        self._err = OracleError
        g = Geometry(**fixture["geometry"])
        self.m = OracleManager(g, **fixture["config"])
        self._cursor = 0

    def init_info(self):
        m = self.m
        return {"buffer_count": m.buffer_count, "groups_per_slot": m.groups_per_slot,
                "slot_stride": m.slot_stride, "buffer_size": m.dev.sizes[0], "init_us": m.init_us}

    def call(self, op, **kw):
        m = self.m
        try:
            if op == "alloc":
                return m.alloc_reqid()
            if op == "free":
                return m.free_reqid(kw["req"])
            if op == "step":
                ok, us = m.step(kw["seq"])
                return [ok, us]
            if op == "plan":
                return m.plan_overlap(kw["seq"])
            if op == "execute":
                return m.execute_plan(kw["plan"])
            if op == "eager":
                return m.eager_prepare(kw["k"])
            if op == "reclaim":
                return list(m.reclaim())
            if op == "reclaim_until":
                return list(m.reclaim_until(kw["target"]))
        except self._err as exc:
            return {"error": exc.kind}
        raise KeyError(op)

    def events(self):
        ev = self.m.dev.events[self._cursor:]
        self._cursor = len(self.m.dev.events)
        return [[0 if k == "map" else 1, b, o] for k, b, o in ev]

    def state(self):
        return self.m.state()


class CoreAdapter:
    """Adapter over the C-ABI allocator core (paper_2405_04437_b200.KVCacheManager).

    backend="shadow" runs the same core without a device (CPU tests); backend="cuda" issues
    every map/unmap to the real driver at 2 MiB (GPU tests)."""

    def __init__(self, fixture, backend="shadow", **mgr_kw):
        from paper_2405_04437_b200 import errors
        from paper_2405_04437_b200.geometry import ModelGeometry
        from paper_2405_04437_b200.manager import KVCacheManager, ManagerConfig

        self._errs = (errors.BatchFullError, errors.DoubleFreeError, ValueError, errors.VmmError)
        g = ModelGeometry(**fixture["geometry"])
        self.m = KVCacheManager(g, ManagerConfig(**fixture["config"]), backend=backend, log_events=True, **mgr_kw)

    def init_info(self):
        m = self.m
        return {"buffer_count": m.buffer_count, "groups_per_slot": m.groups_per_slot,
                "slot_stride": m.slot_stride, "buffer_size": m.buffers[0].size, "init_us": m.init_us}

    def call(self, op, **kw):
        m = self.m
        try:
            if op == "alloc":
                return m.alloc_reqid()
            if op == "free":
                return m.free_reqid(kw["req"])
            if op == "step":
                r = m.step(kw["seq"])
                return [r.ok, r.sync_us]
            if op == "plan":
                return m.plan_overlap(kw["seq"])
            if op == "execute":
                return m.execute_plan(kw["plan"])
            if op == "eager":
                return m.eager_prepare(kw["k"])
            if op == "reclaim":
                return list(m.reclaim())
            if op == "reclaim_until":
                return list(m._reclaim_until(kw["target"]))
        except self._errs as exc:
            return {"error": type(exc).__name__}
        raise KeyError(op)

    def events(self):
        return self.m.drain_events()

    def state(self):
        return self.m.parity_state()

    def close(self):
        self.m.close()


def replay_serving_log(record, geo, page_group_size, pool, eager, threshold):
    """Re-issue a serving.run(record=...) log to oracle/allocator.py in the reference order and
    assert the allocator state after every iteration (see tests/test_gpu_serving_replay.py)."""
    from oracle.allocator import Geometry, OracleManager

    om = OracleManager(Geometry(geo.n_layers, geo.kv_heads_total, geo.head_dim, geo.bytes_per_elem,
                                geo.max_context, geo.max_batch, geo.tp_degree), page_group_size, pool_bytes=pool,
                       reclaim_threshold=threshold, eager_groups=eager)
    stats = {"iterations": 0, "plans": 0, "preemptions": 0, "reclaims": 0}
    for it in record:
        for rid in it["admits"]:
            assert om.alloc_reqid() == rid, (it["it"], "admit")
        if it["bg"]:
            if it["plan"]:
                om.execute_plan([tuple(x) for x in it["plan"]])
                stats["plans"] += 1
            om.eager_prepare()
            freed, _ = om.reclaim()
            stats["reclaims"] += int(freed > 0)
        ok, _ = om.step(it["steps"][0])
        for victim, seq in zip(it["preempted"], it["steps"][1:]):
            assert not ok
            om.free_reqid(victim)
            ok, _ = om.step(seq)
            stats["preemptions"] += 1
        assert ok, (it["it"], "step")
        want = it["state"]
        got = om.state()
        for key in ("slots", "eager_slot", "created", "mapped", "precreated", "calls", "total_mapped_bytes"):
            assert got[key] == want[key], (it["it"], key, got[key], want[key])
        for rid in it["frees"]:
            om.free_reqid(rid)
        stats["iterations"] += 1
    return stats
