"""ORACLE — test infrastructure only, never the product path.

CPU restatement of the reference vAttention allocator policy (`kvsim.manager.KVCacheManager`
over the mock driver `kvsim.vmm.VmmDevice`), written independently from the reference source so
that the GPU box (which has no `/root/reference`) still has a checker.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.

Parity pinning: `tests/golden/make_golden.py` records the *reference itself* (imported from
`/root/reference/pkg/src`) on a set of call scripts; `tests/test_oracle_golden.py` replays those
scripts through this module and demands bit-identical results, event logs, slot tuples, pool
counters, per-API call counts and modelled latencies.

Citations are `/root/reference/pkg/src/kvsim/<file>:<line>`.
"""

from __future__ import annotations

from dataclasses import dataclass

KIB = 1024
MB2 = 2 * KIB * KIB

# Table 2 of the paper, per-call microseconds keyed by page-group size (vmm.py:55-68).
TABLE2_US = {
    "vMemReserve": {65536: 18.0, 131072: 17.0, 262144: 16.0},
    "cuMemAddressReserve": {MB2: 2.0},
    "vMemCreate": {65536: 1.7, 131072: 2.0, 262144: 2.1},
    "cuMemCreate": {MB2: 29.0},
    "vMemMap": {65536: 8.0, 131072: 8.5, 262144: 9.0},
    "cuMemMap": {MB2: 2.0},
    "cuMemSetAccess": {MB2: 38.0},
    "cuMemUnmap": {MB2: 34.0},
    "vMemRelease": {65536: 2.0, 131072: 3.0, 262144: 4.0},
    "cuMemRelease": {MB2: 23.0},
    "vMemFree": {65536: 35.0, 131072: 35.0, 262144: 35.0},
    "cuMemAddressFree": {MB2: 1.0},
}


class OracleError(Exception):
    """Base; `kind` names the reference exception class it stands for."""

    kind = "Error"


class BatchFull(OracleError):
    kind = "BatchFullError"          # manager.py:28


class DoubleFree(OracleError):
    kind = "DoubleFreeError"         # manager.py:32


class BadArgument(OracleError):
    kind = "ValueError"              # manager.py:265-272


class PoolExhausted(OracleError):
    kind = "PoolExhaustedError"      # vmm.py:34


class BadMapping(OracleError):
    kind = "MappingError"            # vmm.py:38


class Misaligned(OracleError):
    kind = "AlignmentError"          # vmm.py:30


class BadFree(OracleError):
    kind = "InvalidFreeError"        # vmm.py:42


def ceil_groups(nbytes: int, t: int) -> int:
    """geometry.py:177-183 — page-groups covering nbytes."""
    if nbytes < 0 or t < 1:
        raise BadArgument("ceil_groups domain")
    return -(-nbytes // t)


@dataclass(frozen=True)
class Geometry:
    """geometry.py:64-117 (only the fields the allocator consumes)."""

    n_layers: int
    kv_heads_total: int
    head_dim: int
    bytes_per_elem: int
    max_context: int
    max_batch: int
    tp_degree: int = 1

    @property
    def token_layer_bytes(self) -> int:        # geometry.py:100-103
        return (self.kv_heads_total // self.tp_degree) * self.head_dim * self.bytes_per_elem


class ShadowDevice:
    """Driver bookkeeping shadow: the mock `VmmDevice` state machine (vmm.py:150-302).

    Buffers are (id -> size, {offset: handle_id}); handles are id -> [state, buffer, offset].
    `events` is the ordered log of ('map'|'unmap', buffer_id, offset) the parity tests compare.
    """

    def __init__(self, capacity: int, t: int, table=None):
        self.capacity, self.t = capacity, t
        self.table = table or TABLE2_US
        self.created = 0
        self.mapped = 0
        self.precreated = 0
        self.total_mapped_bytes = 0
        self.next_handle = 0
        self.sizes: list[int] = []
        self.maps: list[dict[int, int]] = []
        self.handles: dict[int, list] = {}
        self.calls: dict[str, int] = {}
        self.ledger: dict[str, float] = {}
        self.events: list[tuple[str, int, int]] = []
        big = t == MB2                                          # vmm.py:178-182
        self.api_reserve = ("cuMemAddressReserve",) if big else ("vMemReserve",)
        self.api_create = ("cuMemCreate",) if big else ("vMemCreate",)
        self.api_map = ("cuMemMap", "cuMemSetAccess") if big else ("vMemMap",)
        self.api_release = ("cuMemUnmap", "cuMemRelease") if big else ("vMemRelease",)

    # vmm.py:186-195 — each API charged `count` times; the composite is a built-in sum()
    # (compensated summation on CPython >= 3.12, which the C++ core reproduces).
    def _charge_one(self, api, count):
        us = self.table[api][self.t] * count
        self.ledger[api] = self.ledger.get(api, 0.0) + us
        self.calls[api] = self.calls.get(api, 0) + count
        return us

    def bill(self, apis, count: int = 1) -> float:
        return sum(self._charge_one(api, count) for api in apis)

    def unit_cost(self, apis) -> float:
        return sum(self.table[api][self.t] for api in apis)

    @property
    def available(self) -> int:                 # vmm.py:124-127
        return self.capacity - self.mapped * self.t

    @property
    def free(self) -> int:                      # vmm.py:118-121
        return self.capacity - self.created * self.t

    def reserve(self, size: int) -> int:        # vmm.py:199-211
        if size % self.t:
            raise Misaligned(size)
        self.sizes.append(size)
        self.maps.append({})
        self.bill(self.api_reserve)
        return len(self.sizes) - 1

    def _new_handle(self) -> int:
        hid = self.next_handle
        self.next_handle += 1
        self.handles[hid] = ["created", None, None]
        return hid

    def create(self) -> int:                    # vmm.py:213-225
        if self.free < self.t:
            raise PoolExhausted("pool")
        hid = self._new_handle()
        self.created += 1
        self.bill(self.api_create)
        return hid

    def precreate(self, count: int) -> float:   # vmm.py:227-239
        if count < 0:
            raise BadArgument(count)
        if self.free < count * self.t:
            raise PoolExhausted("precreate")
        self.created += count
        self.precreated += count
        return self.bill(self.api_create, count) if count else 0.0

    def take_precreated(self) -> int:           # vmm.py:245-253
        if self.precreated < 1:
            raise PoolExhausted("reserve empty")
        self.precreated -= 1
        return self._new_handle()

    def map(self, buf: int, off: int, hid: int) -> float:   # vmm.py:255-283
        h = self.handles[hid]
        if h[0] != "created":
            raise BadMapping(hid)
        if off % self.t:
            raise Misaligned(off)
        if off < 0 or off + self.t > self.sizes[buf]:
            raise BadMapping(off)
        if off in self.maps[buf]:
            raise BadMapping(off)
        h[0], h[1], h[2] = "mapped", buf, off
        self.maps[buf][off] = hid
        self.mapped += 1
        self.total_mapped_bytes += self.t
        self.events.append(("map", buf, off))
        return self.bill(self.api_map)

    def unmap_release(self, buf: int, off: int) -> float:   # vmm.py:285-297
        if off not in self.maps[buf]:
            raise BadFree(off)
        hid = self.maps[buf].pop(off)
        del self.handles[hid]
        self.mapped -= 1
        self.created -= 1
        self.events.append(("unmap", buf, off))
        return self.bill(self.api_release)

    def charged_total(self) -> float:           # vmm.py:301-302
        return sum(self.ledger.values())


INACTIVE, PREFILL, DECODE = "inactive", "prefill", "decode"


class OracleManager:
    """Restatement of the vAttention allocator policy (manager.py:84-372).

    Per slot we keep [active, context_len, mapped_groups, phase, freed_seq] (manager.py:66-75).
    """

    def __init__(self, g: Geometry, page_group_size: int, pool_bytes: int = 80 * KIB ** 3,
                 reclaim_threshold: float = 0.10, eager_groups: int = 0, sliced: bool = False,
                 pre_create_fraction: float = 1.0, table=None):
        if not 0.0 <= reclaim_threshold <= 1.0 or not 0.0 <= pre_create_fraction <= 1.0:
            raise BadArgument("fraction")                       # manager.py:56-63
        if eager_groups < 0:
            raise BadArgument("eager_groups")
        if g.max_batch < 1:                                     # manager.py:86-87
            raise BadArgument("max_batch")
        t = int(page_group_size)
        self.g, self.t = g, t
        self.pool_bytes = pool_bytes
        self.reclaim_threshold = reclaim_threshold
        self.eager_groups = eager_groups
        # manager.py:93-99 — 2N per-layer buffers, or 2 layer-sliced ones
        self.buffer_count = 2 if sliced else 2 * g.n_layers
        self.token_bytes = g.token_layer_bytes * (g.n_layers if sliced else 1)
        if t < self.token_bytes:                                # manager.py:100-104
            raise BadArgument("page group below one token")
        if pool_bytes < self.buffer_count * t:                  # manager.py:105-109
            raise BadArgument("pool below one group per buffer")
        self.groups_per_slot = ceil_groups(g.max_context * self.token_bytes, t)   # :111-115
        self.slot_stride = self.groups_per_slot * t
        self.dev = ShadowDevice(pool_bytes, t, table)
        for _ in range(self.buffer_count):                      # :119-122
            self.dev.reserve(g.max_batch * self.slot_stride)
        self.init_us = self.dev.charged_total()
        self.init_us += self.dev.precreate(int(pre_create_fraction * pool_bytes) // t)   # :124-125
        self.slots = [[False, 0, 0, INACTIVE, 0] for _ in range(g.max_batch)]
        self.eager_slot = None
        self.freed_counter = 0
        self.rollback: list[int] = []                           # manager.py:130 _handle_cache

    # -- sizing (manager.py:134-138) --
    def groups_required(self, seq_len: int) -> int:
        return ceil_groups(seq_len * self.token_bytes, self.t)

    def offset(self, rid: int, gi: int) -> int:
        return rid * self.slot_stride + gi * self.t

    def floor(self) -> int:                                     # manager.py:157-158
        return int(self.reclaim_threshold * self.pool_bytes)

    def _best_inactive(self):
        """argmax over inactive slots of (mapped_groups, -req_id) (manager.py:171-174, :349)."""
        best = None
        for rid, s in enumerate(self.slots):
            if s[0]:
                continue
            if best is None or s[2] > self.slots[best][2]:
                best = rid
        return best

    # -- lifecycle (manager.py:163-190) --
    def alloc_reqid(self) -> int:
        es = self.eager_slot
        if es is not None and not self.slots[es][0]:
            rid = es
            self.eager_slot = None
        else:
            rid = self._best_inactive()
            if rid is None:
                raise BatchFull("all slots active")
        s = self.slots[rid]
        s[0], s[1], s[3] = True, 0, PREFILL
        return rid

    def free_reqid(self, rid: int) -> None:
        s = self.slots[rid]
        if not s[0]:
            raise DoubleFree(rid)
        self.freed_counter += 1
        s[0], s[1], s[3], s[4] = False, 0, INACTIVE, self.freed_counter

    # -- mapping machinery (manager.py:194-251) --
    def _grab_handle(self):
        if self.rollback:
            return self.rollback.pop(0), 0.0
        if self.dev.precreated:
            return self.dev.take_precreated(), 0.0
        hid = self.dev.create()
        return hid, self.dev.unit_cost(self.dev.api_create)

    def _map_group(self, rid: int, gi: int) -> float:
        got, us = [], 0.0
        try:
            for _ in range(self.buffer_count):
                hid, c = self._grab_handle()
                got.append(hid)
                us += c
        except PoolExhausted:
            self.rollback.extend(got)
            raise
        off = self.offset(rid, gi)
        for buf, hid in enumerate(got):
            us += self.dev.map(buf, off, hid)
        return us

    def _drop_top(self, rid: int) -> float:
        s = self.slots[rid]
        gi = s[2] - 1
        us = 0.0
        off = self.offset(rid, gi)
        for buf in range(self.buffer_count):
            us += self.dev.unmap_release(buf, off)
        s[2] = gi
        return us

    def victims(self):
        order = [r for r, s in enumerate(self.slots) if not s[0] and s[2] > 0]
        order.sort(key=lambda r: (r == self.eager_slot, self.slots[r][4], r))
        return order

    def reclaim_until(self, target: int):
        freed, us = 0, 0.0
        for rid in self.victims():
            s = self.slots[rid]
            while s[2] > 0 and self.dev.available < target:
                us += self._drop_top(rid)
                freed += 1
            if s[2] == 0 and self.eager_slot == rid:
                self.eager_slot = None
            if self.dev.available >= target:
                break
        return freed, us

    # -- iteration entry points (manager.py:255-372) --
    def step(self, seq_lens):
        if len(seq_lens) != len(self.slots):
            raise BadArgument("length")
        for rid, s in enumerate(self.slots):
            n = seq_lens[rid]
            if not s[0] and n != 0:
                raise BadArgument("inactive nonzero")
            if n < 0 or n > self.g.max_context:
                raise BadArgument("range")
        sync = 0.0
        for rid, s in enumerate(self.slots):
            if not s[0]:
                continue
            need = self.groups_required(seq_lens[rid])
            if s[3] == PREFILL:
                while s[2] > need:
                    sync += self._drop_top(rid)
            while s[2] < need:
                try:
                    sync += self._map_group(rid, s[2])
                except PoolExhausted:
                    freed, rus = self.reclaim_until(self.buffer_count * self.t)
                    sync += rus
                    if freed == 0:
                        return False, sync
                    continue
                s[2] += 1
            s[1], s[3] = seq_lens[rid], DECODE
        return True, sync

    def plan_overlap(self, next_lens):
        plan = []
        for rid, s in enumerate(self.slots):
            if not s[0]:
                continue
            top = min(self.groups_required(next_lens[rid]), self.groups_per_slot)
            for gi in range(s[2], top):
                off = self.offset(rid, gi)
                plan.extend((rid, b, off) for b in range(self.buffer_count))
        return plan

    def execute_plan(self, plan) -> float:
        us, seen = 0.0, set()
        for rid, _buf, off in plan:
            s = self.slots[rid]
            gi = (off - rid * self.slot_stride) // self.t
            if (rid, gi) in seen or gi < s[2] or gi >= self.groups_per_slot:
                continue
            while s[2] <= gi:
                try:
                    us += self._map_group(rid, s[2])
                except PoolExhausted:
                    return us
                s[2] += 1
            seen.add((rid, gi))
        return us

    def eager_prepare(self, k=None) -> float:
        k = self.eager_groups if k is None else k
        if k <= 0:
            return 0.0
        k = min(k, self.groups_per_slot)
        es = self.eager_slot
        if es is not None and self.slots[es][2] >= k:
            return 0.0
        rid = self._best_inactive()
        if rid is None:
            return 0.0
        self.eager_slot = rid
        s = self.slots[rid]
        us = 0.0
        group_bytes = self.buffer_count * self.t
        while s[2] < k:
            if self.dev.available - group_bytes < self.floor():
                break
            try:
                us += self._map_group(rid, s[2])
            except PoolExhausted:
                break
            s[2] += 1
        return us

    def reclaim(self):
        fl = self.floor()
        if self.dev.available >= fl:
            return 0, 0.0
        return self.reclaim_until(fl)

    # -- state export for parity comparisons --
    def state(self) -> dict:
        return {
            "slots": [[int(s[0]), s[1], s[2], s[3], s[4]] for s in self.slots],
            "eager_slot": self.eager_slot,
            "created": self.dev.created,
            "mapped": self.dev.mapped,
            "precreated": self.dev.precreated,
            "calls": dict(sorted(self.dev.calls.items())),
            "total_mapped_bytes": self.dev.total_mapped_bytes,
            "charged_us": self.dev.charged_total(),
        }
