"""Algorithm-1 serving loop over the vAttention allocator.

The event order is the reference simulator's (kvsim/simulator.py:333-504): admit arrivals ->
background allocation work (overlapped mode: execute_plan -> eager_prepare -> reclaim) -> step
(preempting the newest request on failure) -> compute -> plan the next iteration's decode growth
-> retire finished requests.  Two clocks:

* ``clock="model"`` advances time with the reference's linear IterationModel and the modelled
  Table-2 latencies, so the per-iteration records equal ``kvsim.simulator.run`` exactly
  (tests/test_serving_parity.py) while the allocator calls go through the C++ core;
* ``clock="wall"`` runs the real sm_100a kernels per iteration (KV append + prefill attention
  for new requests, KV append + decode attention for the batch) on the real cuMem* backend and
  measures, per iteration, the host time the allocator keeps off the GPU ("exposed map ms").

Overlapped mode runs the planned maps on the background thread *during* the iteration's
kernels (submitted right after launch, with plan credits so admission ranks slots exactly as
the reference does), and queues eager_prepare/reclaim behind step whenever that provably
yields the same state (vattn_iteration_step, VATTN_ITER_DEFER).
"""

from __future__ import annotations

import csv
import json
import time
from collections import deque
from dataclasses import dataclass, field

from .errors import BatchFullError
from .manager import KVCacheManager, ManagerConfig

MB2 = 2 * 1024 * 1024


class SimulationAborted(RuntimeError):
    """No forward progress within the preemption cap (simulator.py:40-41)."""


@dataclass(frozen=True)
class IterationModel:
    """Linear compute proxy of the reference (simulator.py:45-62); model clock only."""

    c0_ms: float = 10.0
    c1_ms_per_token: float = 0.0005

    def compute_ms(self, tokens: int) -> float:
        return self.c0_ms + self.c1_ms_per_token * tokens


class GemmDense:
    """Dense layers of an iteration (QKV/O projections, MLP) as real bf16 GEMMs on the GPU, sized
    to the reference IterationModel's duration (simulator.py:45-62): each unit multiplies a
    [1024, 8192] activation by one of 8 distinct [8192, 8192] weight matrices (137 GFLOP and 128 MiB
    of weights per unit, 1 GiB per cycle through the 8), so the attention kernels and the
    allocator's driver calls see real tensor-core and HBM contention instead of an idle sleep.  Calibrated once at
    construction (median unit time on this GPU).  cuBLAS, not a product kernel."""

    def __init__(self, model: "IterationModel | None" = None, device: int = 0, n_weights: int = 8,
                 dim: int = 8192, rows: int = 1024):
        import torch

        self.model = model or IterationModel()
        dev = torch.device("cuda", device)
        gen = torch.Generator(device=dev).manual_seed(1)
        self.w = [torch.randn(dim, dim, device=dev, generator=gen, dtype=torch.bfloat16) * 0.01
                  for _ in range(n_weights)]
        self.x = torch.randn(rows, dim, device=dev, generator=gen, dtype=torch.bfloat16)
        self.y = torch.empty(rows, dim, device=dev, dtype=torch.bfloat16)
        self.i = 0
        for _ in range(3):
            self._unit()
        torch.cuda.synchronize(dev)
        times = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(16):
                self._unit()
            e1.record()
            torch.cuda.synchronize(dev)
            times.append(e0.elapsed_time(e1) / 16)
        self.unit_ms = sorted(times)[len(times) // 2]
        self.launches = 0

    def _unit(self):
        import torch

        torch.matmul(self.x, self.w[self.i % len(self.w)], out=self.y)
        self.i += 1

    def compute_ms(self, tokens: int) -> float:
        return self.model.compute_ms(tokens)

    def launch(self, tokens: int) -> int:
        """Enqueue GEMM units totalling ~compute_ms(tokens) on the current stream."""
        n = max(1, round(self.compute_ms(tokens) / self.unit_ms))
        for _ in range(n):
            self._unit()
        self.launches += n
        return n


@dataclass
class IterationRecord:
    iteration: int
    end_ms: float
    batch: int
    prefills: int
    tokens: int
    compute_ms: float
    sync_alloc_ms: float
    stall_ms: float
    cpu_ms: float
    committed_bytes: int
    used_bytes: int
    alloc_bytes: int
    preemptions: int
    # measured (wall clock); zero under the model clock
    exposed_ms: float = 0.0
    kernel_ms: float = 0.0
    bg_wall_ms: float = 0.0
    deferred: int = 0
    # real driver activity during this iteration (CUDA backend)
    drv_maps: int = 0
    drv_unmaps: int = 0
    drv_set_access_ms: float = 0.0
    drv_unmap_ms: float = 0.0
    drv_create_ms: float = 0.0
    t_admit_ms: float = 0.0
    t_bgwait_ms: float = 0.0
    t_step_ms: float = 0.0
    t_retire_ms: float = 0.0
    # physically mapped bytes (logical + speculative/lazily kept pages, or whole chunks with
    # phys_chunk_groups > 1); equals committed_bytes on the model clock
    phys_bytes: int = 0

    REF_FIELDS = ("iteration", "end_ms", "batch", "prefills", "tokens", "compute_ms", "sync_alloc_ms",
                  "stall_ms", "cpu_ms", "committed_bytes", "used_bytes", "alloc_bytes", "preemptions")
    CSV_FIELDS = REF_FIELDS + ("exposed_ms", "kernel_ms", "bg_wall_ms", "deferred", "drv_maps", "drv_unmaps",
                               "drv_set_access_ms", "drv_unmap_ms", "drv_create_ms", "t_admit_ms",
                               "t_bgwait_ms", "t_step_ms", "t_retire_ms", "phys_bytes")

    def row(self, fields=CSV_FIELDS) -> list:
        return [getattr(self, f) for f in fields]


@dataclass
class ServingMetrics:
    iterations: list = field(default_factory=list)
    completed_requests: int = 0
    generated_tokens: int = 0
    preemptions: int = 0
    init_alloc_ms: float = 0.0
    init_wall_ms: float = 0.0
    # per request (trace index): arrival, first admission and first-token times (clock ms); the
    # first token of a request is produced by the iteration that runs its prefill
    req_arrival_ms: dict = field(default_factory=dict)
    req_admit_ms: dict = field(default_factory=dict)
    req_first_token_ms: dict = field(default_factory=dict)

    def request_summary(self) -> dict:
        """Time to first token and queueing delay (admission - arrival), ms: what staged admission
        or a stalled iteration costs a request (not in the reference's summary)."""
        ttft = [self.req_first_token_ms[i] - self.req_arrival_ms[i] for i in self.req_first_token_ms]
        queue = [self.req_admit_ms[i] - self.req_arrival_ms[i] for i in self.req_admit_ms]
        out = {"requests_with_first_token": len(ttft)}
        for name, v in (("ttft_ms", ttft), ("queue_ms", queue)):
            out[f"{name}_mean"] = sum(v) / len(v) if v else 0.0
            out[f"{name}_p50"] = self._pct(v, 0.50)
            out[f"{name}_p99"] = self._pct(v, 0.99)
            out[f"{name}_max"] = max(v, default=0.0)
        return out

    @staticmethod
    def _pct(values, q):
        if not values:
            return 0.0
        v = sorted(values)
        rank = -(-q * len(v) // 1)
        return v[min(len(v), max(1, int(rank))) - 1]

    def summary(self) -> dict:
        """Same keys as SimMetrics.summary (simulator.py:118-141) + measured exposure."""
        its = self.iterations
        lat = [r.compute_ms + r.stall_ms + r.cpu_ms for r in its]
        end = its[-1].end_ms if its else 0.0
        n = len(its)
        out = {
            "iterations": n,
            "max_batch": max((r.batch for r in its), default=0),
            "completed_requests": self.completed_requests,
            "generated_tokens": self.generated_tokens,
            "tokens_per_s": self.generated_tokens / (end / 1000.0) if end > 0 else 0.0,
            "sim_time_ms": end,
            "p50_iteration_ms": self._pct(lat, 0.50),
            "p99_iteration_ms": self._pct(lat, 0.99),
            "stall_ms_total": sum(r.stall_ms for r in its),
            "sync_alloc_ms_total": sum(r.sync_alloc_ms for r in its),
            "cpu_ms_total": sum(r.cpu_ms for r in its),
            "preemptions": self.preemptions,
            "peak_committed_bytes": max((r.committed_bytes for r in its), default=0),
            "peak_used_bytes": max((r.used_bytes for r in its), default=0),
            "mean_waste_bytes": sum(r.committed_bytes - r.used_bytes for r in its) / n if n else 0.0,
            "mean_phys_waste_bytes": sum(max(r.phys_bytes, r.committed_bytes) - r.used_bytes for r in its) / n if n else 0.0,
            "peak_phys_bytes": max((max(r.phys_bytes, r.committed_bytes) for r in its), default=0),
            "init_alloc_ms": self.init_alloc_ms,
        }
        ex = [r.exposed_ms for r in its]
        out.update({
            "exposed_map_ms_per_iter": sum(ex) / n if n else 0.0,
            "exposed_map_ms_p99": self._pct(ex, 0.99),
            "exposed_map_ms_max": max(ex, default=0.0),
            "kernel_ms_total": sum(r.kernel_ms for r in its),
            "init_wall_ms": self.init_wall_ms,
        })
        out.update(self.request_summary())
        return out

    def write_iterations_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(IterationRecord.CSV_FIELDS)
            for r in self.iterations:
                w.writerow(r.row())

    def write_summary_json(self, path) -> None:
        with open(path, "w") as fh:
            json.dump(self.summary(), fh, indent=2, sort_keys=True)
            fh.write("\n")


@dataclass
class _Running:
    record_index: int
    prompt_tokens: int
    decode_tokens: int
    ctx: int
    produced: int = 0
    admit_order: int = 0


class SyntheticModel:
    """Attention-only model forward on the virtual KV cache: per layer KV-append of this
    iteration's tokens, prefill attention for newly admitted requests and one batched decode
    attention for the rest.  Inputs are seeded random bf16 (no weights: the hot path under test
    is the KV cache and attention)."""

    def __init__(self, mgr: KVCacheManager, geometry, max_prompt: int, seed: int = 0,
                 dense_model: "IterationModel | None" = None):
        import torch

        self.t = torch
        self.mgr = mgr
        g = geometry
        self.layers = g.n_layers
        self.hq, self.hkv, self.d = g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim
        self.dev = torch.device("cuda", mgr.device)
        gen = torch.Generator(device=self.dev).manual_seed(seed)
        B = g.max_batch
        self.q_pf = torch.randn(max_prompt, self.hq, self.d, device=self.dev, generator=gen, dtype=torch.bfloat16)
        self.k_pf = torch.randn(1, max_prompt, self.hkv, self.d, device=self.dev, generator=gen, dtype=torch.bfloat16)
        self.v_pf = torch.randn_like(self.k_pf)
        self.q_dec = torch.randn(B, self.hq, self.d, device=self.dev, generator=gen, dtype=torch.bfloat16)
        self.k_dec = torch.randn(B, self.hkv, self.d, device=self.dev, generator=gen, dtype=torch.bfloat16)
        self.v_dec = torch.randn_like(self.k_dec)
        self.out_pf = torch.empty_like(self.q_pf)
        self.out_dec = torch.empty_like(self.q_dec)
        self.zero = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.dense_model = dense_model
        self.q_pack = None           # packed queries of an iteration's prompts (varlen prefill)
        self.out_pack = None

    def forward(self, prefills, decodes) -> None:
        """prefills: [(slot, prompt_len)]; decodes: [(slot, ctx)] (ctx includes the new token)."""
        from .attention import decode_attention_append, kv_append, prefill_attention, prefill_attention_varlen

        t = self.t
        dense_tokens = sum(n for _, n in prefills) + len(decodes)
        if len(prefills) > 1:   # all new prompts' attention in one varlen launch per layer
            lens = [n for _, n in prefills]
            total = sum(lens)
            if self.q_pack is None or self.q_pack.shape[0] < total:
                self.q_pack = t.randn(total, self.hq, self.d, device=self.dev, dtype=t.bfloat16)
                self.out_pack = t.empty_like(self.q_pack)
            idxs = [t.tensor([slot], dtype=t.int32, device=self.dev) for slot, _ in prefills]
            for layer in range(self.layers):
                for (slot, n), idx in zip(prefills, idxs):
                    kv_append(self.mgr, layer, self.k_pf[:, :n], self.v_pf[:, :n], self.zero, idx)
                prefill_attention_varlen(self.mgr, layer, self.q_pack[:total], lens, [s_ for s_, _ in prefills],
                                         out=self.out_pack[:total])
            prefills = []
        for slot, n in prefills:
            idx = t.tensor([slot], dtype=t.int32, device=self.dev)
            for layer in range(self.layers):
                kv_append(self.mgr, layer, self.k_pf[:, :n], self.v_pf[:, :n], self.zero, idx)
                prefill_attention(self.mgr, layer, self.q_pf[:n], slot, kv_len=n, out=self.out_pf[:n])
        if decodes:
            B = len(decodes)
            idx = t.tensor([s for s, _ in decodes], dtype=t.int32, device=self.dev)
            before = t.tensor([c - 1 for _, c in decodes], dtype=t.int32, device=self.dev)
            for layer in range(self.layers):   # fused: append row ctx-1 and attend over ctx rows
                decode_attention_append(self.mgr, layer, self.q_dec[:B], self.k_dec[:B], self.v_dec[:B],
                                        before, idx, out=self.out_dec[:B])
        if self.dense_model is not None:
            # the dense layers (QKV/O projections, MLP) of the iteration, as device time: real
            # GEMMs (GemmDense) or the calibrated sleep kernel (IterationModel)
            tokens = dense_tokens
            if hasattr(self.dense_model, "launch"):
                self.dense_model.launch(tokens)
            else:
                import ctypes as C

                from ._abi import check, lib
                ns = int(self.dense_model.compute_ms(tokens) * 1e6)
                check(lib().vattn_compute_proxy(ns, C.c_void_p(t.cuda.current_stream().cuda_stream)))


def median_prompt_groups(records, geometry, page_group_size: int, sliced: bool = False) -> int:
    """Default eager page-groups = groups covering the median prompt (simulator.py:507-520)."""
    if not records:
        return 0
    prompts = sorted(r[1] for r in records)
    median = prompts[(len(prompts) - 1) // 2]
    tb = geometry.per_token_layer_bytes * (geometry.n_layers if sliced else 1)
    return -(-median * tb // int(page_group_size))


def load_trace_csv(path) -> list[tuple[int, int, int]]:
    with open(path, newline="") as fh:
        rd = csv.reader(fh)
        next(rd)
        return [(int(a), int(p), int(d)) for a, p, d in rd if a]


def run(records, geometry, *, mode: str = "overlapped", clock: str = "model",
        page_group_size: int = MB2, pool_bytes: int = 80 * 1024 ** 3, reclaim_threshold: float = 0.10,
        eager_groups: int = 0, sliced: bool = False, pre_create_fraction: float = 1.0,
        iteration_model: IterationModel | None = None, preemption_cap: int = 1000,
        backend: str | None = None, defer: bool | None = None, observer=None,
        max_iterations: int | None = None, model: SyntheticModel | None = None,
        manager: KVCacheManager | None = None, dense_proxy: IterationModel | None = None,
        prefetch_tokens: int = 0, prefetch_slots: int = 0, prefetch_slot_tokens: int = 0,
        lazy_unmap: bool = False, stage_admission: bool = False, stage_max_iters: int = 8,
        hold_worker: bool = False, record: list | None = None, phys_chunk_groups: int = 1) -> ServingMetrics:
    """Replay `records` = [(arrival_ms, prompt_tokens, decode_tokens)] (trace.py:26-31).

    B200 additions (wall clock, CUDA backend; the allocator's logical state stays the
    reference's for the calls made): `lazy_unmap` keeps trimmed/reclaimed pages mapped until
    their handle is needed; `stage_admission` holds an arrived request at the head of the queue
    (FIFO kept) until the slot alloc_reqid will give it has its prompt pages mapped by the
    prefetch worker, for at most `stage_max_iters` iterations and never while the batch is
    empty, so prompt mapping overlaps the running batch's compute instead of stalling it.
    `phys_chunk_groups` backs that many consecutive page-groups of a buffer with one physical
    handle (one cuMemMap + cuMemSetAccess per chunk; bookkeeping still per 2 MiB group).

    `record` (a list): append one entry per iteration with the logical allocator calls in the
    reference's order (admits, the plan executed for this iteration, eager/reclaim, the step
    arguments, preemptions, frees) and the allocator state after the step
    (`parity_state()`, joining the background thread), for replay through the oracle
    (tests/test_gpu_serving_replay.py)."""
    if mode not in ("sync", "overlapped"):
        raise ValueError(f"mode must be 'sync' or 'overlapped', got {mode!r}")
    if clock not in ("model", "wall"):
        raise ValueError(f"clock must be 'model' or 'wall', got {clock!r}")
    for i, (_, p, d) in enumerate(records):
        if p + d > geometry.max_context:
            raise ValueError(f"trace record {i}: prompt+decode ({p}+{d}) exceeds max_context")
    wall = clock == "wall"
    if defer is None:
        defer = wall               # model clock keeps the reference's exact call order
    im = iteration_model or IterationModel()
    own_manager = manager is None
    mgr = manager or KVCacheManager(
        geometry, ManagerConfig(page_group_size=int(page_group_size), pool_bytes=pool_bytes,
                                reclaim_threshold=reclaim_threshold, eager_groups=eager_groups,
                                sliced=sliced, pre_create_fraction=pre_create_fraction),
        backend=backend or ("cuda" if wall else "shadow"), prefetch_tokens=prefetch_tokens,
        prefetch_slots=prefetch_slots, prefetch_slot_tokens=prefetch_slot_tokens, lazy_unmap=lazy_unmap,
        phys_chunk_groups=phys_chunk_groups)
    stage = bool(stage_admission) and wall and mode == "overlapped"
    staged_iters: dict[int, int] = {}     # record index -> iterations held at the queue head
    if wall and model is None:
        model = SyntheticModel(mgr, geometry, max(p for _, p, _ in records) if records else 1,
                               dense_model=dense_proxy)
    if wall:
        import torch

    metrics = ServingMetrics(init_alloc_ms=mgr.init_us / 1000.0, init_wall_ms=mgr.init_wall_us / 1000.0)
    token_bytes = 2 * geometry.n_layers * geometry.per_token_layer_bytes
    pending: deque = deque(enumerate(records))
    running: dict[int, _Running] = {}
    seq_lens = [0] * geometry.max_batch
    clock_us = 0
    iteration = 0
    admit_counter = 0
    prev_compute_budget_us = 0.0
    prev_alloc_cum = mgr.vmm.total_mapped_bytes
    t_start = time.perf_counter()
    overlapped = mode == "overlapped"
    drv_prev = mgr.driver_stats(peek=True) if wall else None

    prev_plan = None
    while pending or running:
        if max_iterations is not None and iteration >= max_iterations:
            break
        rec_it = {"it": iteration, "admits": [], "plan": prev_plan, "bg": overlapped, "steps": [],
                  "preempted": [], "frees": []} if record is not None else None
        t_it = time.perf_counter()
        if wall:
            clock_us = max(clock_us, int((t_it - t_start) * 1e6))
        if not running and pending:
            clock_us = max(clock_us, pending[0][1][0] * 1000)
            if wall:      # idle: let real time catch up with the next arrival
                gap = clock_us / 1e6 - (time.perf_counter() - t_start)
                if gap > 0:
                    time.sleep(gap)
        # -- admit (Algorithm 1 lines 6-11) --
        t_exp = time.perf_counter()
        while pending and pending[0][1][0] * 1000 <= clock_us:
            if stage and running:
                head_index, head_rec = pending[0]
                pred = mgr.predict_alloc(1)
                if pred and not mgr.slot_ready(pred[0], head_rec[1]):
                    waited = staged_iters.get(head_index, 0)
                    if waited < stage_max_iters:
                        staged_iters[head_index] = waited + 1
                        break
            try:
                rid = mgr.alloc_reqid()
            except BatchFullError:
                break
            index, rec = pending.popleft()
            running[rid] = _Running(index, rec[1], rec[2], ctx=rec[1], admit_order=admit_counter)
            admit_counter += 1
            seq_lens[rid] = rec[1]
            metrics.req_arrival_ms.setdefault(index, float(rec[0]))
            metrics.req_admit_ms.setdefault(index, clock_us / 1000.0)
            if record is not None:
                rec_it["admits"].append(rid)
        if not running and pending:
            raise SimulationAborted("no request can be admitted into an empty batch")
        t_adm = time.perf_counter()
        # -- background work + step (line 13) --
        bg_us = 0.0
        bg_wall_ms = 0.0
        deferred = 0
        if overlapped:
            bgr = mgr.bg_wait()                  # the plan executed during the previous compute
            bg_wall_ms = bgr.bg_wall_us / 1000.0
        t_bgw = time.perf_counter()
        if overlapped:
            it_res = mgr.iteration_step(seq_lens, eager=True, reclaim=True, defer=defer)
            bg_us = bgr.plan_us + bgr.eager_us + bgr.reclaim_us + it_res.eager_us + it_res.reclaim_us
            ok, us = it_res.ok, it_res.sync_us
            deferred = int(it_res.deferred)
        else:
            r = mgr.step(seq_lens)
            ok, us = r.ok, r.sync_us
        if record is not None:
            rec_it["steps"].append(list(seq_lens))
        overflow_us = max(0.0, bg_us - prev_compute_budget_us)
        sync_us = us
        t_stp = time.perf_counter()
        preempted_here = 0
        while not ok:
            if not running:
                raise SimulationAborted("memory demand cannot be met with an empty batch")
            victim = max(running, key=lambda r: running[r].admit_order)
            state = running.pop(victim)
            mgr.free_reqid(victim)
            seq_lens[victim] = 0
            pending.appendleft((state.record_index, records[state.record_index]))
            preempted_here += 1
            metrics.preemptions += 1
            if metrics.preemptions > preemption_cap:
                raise SimulationAborted(f"aborted after {metrics.preemptions} preemptions")
            r = mgr.step(seq_lens)
            ok = r.ok
            sync_us += r.sync_us
            if record is not None:
                rec_it["preempted"].append(victim)
                rec_it["steps"].append(list(seq_lens))
        if observer is not None:
            observer(mgr, list(seq_lens), iteration)
        if record is not None:
            rec_it["state"] = mgr.parity_state()
            record.append(rec_it)

        batch = len(running)
        tokens = sum(seq_lens[rid] for rid in running)
        prefills = sum(1 for r in running.values() if r.produced == 0)
        # quiescent-point counters (before this iteration's plan starts mapping in background).
        # Wall clock: peek, so a deferred eager/reclaim job keeps running behind the kernels.
        if wall:
            cnt = mgr.peek_counters()
            alloc_cum, committed = cnt.total_mapped_bytes, cnt.mapped * cnt.page_group_size
            phys = cnt.phys_mapped_bytes
        else:
            alloc_cum = mgr.vmm.total_mapped_bytes
            committed = mgr.committed_bytes()
            phys = committed
        exposed_ms = (time.perf_counter() - t_exp) * 1e3
        # -- compute (line 14) + overlapped planning of the next iteration's maps --
        kernel_ms = 0.0
        if wall and batch:
            t_k = time.perf_counter()
            if hold_worker:
                mgr.foreground(True)     # no prefetch driver call during the launch burst
            model.forward([(rid, seq_lens[rid]) for rid, r in running.items() if r.produced == 0],
                          [(rid, seq_lens[rid]) for rid, r in running.items() if r.produced > 0])
            mgr.mark_use()
            if hold_worker:
                mgr.foreground(False)
        if overlapped:
            next_seq = list(seq_lens)
            for rid in running:
                next_seq[rid] = min(seq_lens[rid] + 1, geometry.max_context)
            plan = mgr.plan_overlap(next_seq)
            if record is not None:
                prev_plan = [list(t_) for t_ in plan]
            if stage:
                # prompts that have arrived -> the slots alloc_reqid would give them now; the
                # prefetch worker backs them during these kernels (state is owned here: no join)
                now_ms = (time.perf_counter() - t_start) * 1e3
                arrived = [rec for _, rec in list(pending)[:geometry.max_batch] if rec[0] <= now_ms]
                slots = mgr.predict_alloc(len(arrived)) if arrived else []
                mgr.prefetch_hint(slots, [rec[1] for rec in arrived[:len(slots)]])
            # maps run on the bg thread during the kernels (+ physical prefetch further ahead)
            mgr.bg_submit(plan, credit=True, prefetch=prefetch_tokens > 0 or prefetch_slots > 0 or stage)
        if wall and batch:
            torch.cuda.synchronize()
            kernel_ms = (time.perf_counter() - t_k) * 1e3
        compute_ms = (kernel_ms if wall else im.compute_ms(tokens)) if batch else 0.0
        stall_us = (exposed_ms * 1000.0) if wall else (sync_us + overflow_us)
        if wall:
            clock_us = int((time.perf_counter() - t_start) * 1e6)
        else:
            clock_us += round(compute_ms * 1000) + round(stall_us)
        metrics.iterations.append(IterationRecord(
            iteration=iteration, end_ms=clock_us / 1000.0, batch=batch, prefills=prefills, tokens=tokens,
            compute_ms=compute_ms, sync_alloc_ms=sync_us / 1000.0, stall_ms=stall_us / 1000.0, cpu_ms=0.0,
            committed_bytes=committed, used_bytes=tokens * token_bytes, alloc_bytes=alloc_cum - prev_alloc_cum,
            preemptions=preempted_here, exposed_ms=exposed_ms if wall else 0.0, kernel_ms=kernel_ms,
            bg_wall_ms=bg_wall_ms, deferred=deferred, phys_bytes=phys))
        if wall:
            drv = mgr.driver_stats(peek=True)
            rec = metrics.iterations[-1]
            rec.drv_maps = drv["real_maps"] - drv_prev["real_maps"]
            rec.drv_unmaps = drv["real_unmaps"] - drv_prev["real_unmaps"]
            rec.drv_set_access_ms = (drv["real_set_access_wall_us"] - drv_prev["real_set_access_wall_us"]) / 1e3
            rec.drv_unmap_ms = (drv["real_unmap_wall_us"] - drv_prev["real_unmap_wall_us"]) / 1e3
            rec.drv_create_ms = (drv["real_create_wall_us"] - drv_prev["real_create_wall_us"]) / 1e3
            drv_prev = drv
        prev_alloc_cum = alloc_cum
        prev_compute_budget_us = compute_ms * 1000.0
        # -- retire (lines 15-22); free_reqid waits for deferred eager/reclaim: that is exposed too --
        t_ret = time.perf_counter()
        for rid in list(running):
            st = running[rid]
            if st.produced == 0:
                metrics.req_first_token_ms.setdefault(st.record_index, clock_us / 1000.0)
            st.produced += 1
            if st.produced >= st.decode_tokens:
                metrics.completed_requests += 1
                metrics.generated_tokens += st.decode_tokens
                mgr.free_reqid(rid)
                if record is not None:
                    rec_it["frees"].append(rid)
                seq_lens[rid] = 0
                del running[rid]
            else:
                st.ctx += 1
                seq_lens[rid] = st.ctx
        if wall:
            post = (time.perf_counter() - t_ret) * 1e3
            rec = metrics.iterations[-1]
            rec.exposed_ms += post
            rec.stall_ms += post
            rec.t_admit_ms = (t_adm - t_exp) * 1e3
            rec.t_bgwait_ms = (t_bgw - t_adm) * 1e3
            rec.t_step_ms = (t_stp - t_bgw) * 1e3
            rec.t_retire_ms = post
        iteration += 1
    if overlapped:
        mgr.bg_wait()
    if own_manager:
        if wall:
            import torch
            torch.cuda.synchronize()
            model = None
        mgr.close()              # release the physical pool now, not at garbage collection
    return metrics


# ----------------------------------------------------------------------------- paged comparison
class _BlockPool:
    """PagedAttention-style block allocator (the reference's PagedBlockAllocator semantics,
    kvsim/baselines.py:57-98): one logical block id covers `block_size` tokens of every layer;
    requests grow block by block and free everything on completion."""

    def __init__(self, total_blocks: int, block_size: int):
        self.free = deque(range(total_blocks))
        self.block_size = block_size
        self.owned: dict[int, list[int]] = {}

    def grow(self, rid: int, tokens: int) -> bool:
        need = -(-tokens // self.block_size) - len(self.owned.setdefault(rid, []))
        if need > len(self.free):
            return False
        for _ in range(max(0, need)):
            self.owned[rid].append(self.free.popleft())
        return True

    def release(self, rid: int) -> None:
        self.free.extend(self.owned.pop(rid, []))


def run_paged(records, geometry, *, block_size: int = 16, pool_bytes: int = 24 * 1024 ** 3,
              dense_proxy: IterationModel | None = None, preemption_cap: int = 100_000,
              device: int = 0) -> ServingMetrics:
    """Algorithm-1 loop on the PagedAttention layout with the in-repo paged kernels (config-5
    comparison): per iteration the block tables of the running requests are built on the host and
    uploaded ("block-table preparation"), then paged append / prefill / decode run.
    `exposed_ms` = host time outside the kernels (block allocation + table preparation + upload)."""
    import ctypes as C

    import numpy as np
    import torch

    from ._abi import check, lib
    from .attention import decode_attention_paged, kv_append_paged, prefill_attention_paged

    dev = torch.device("cuda", device)
    g = geometry
    L, hq, hkv, d = g.n_layers, g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim
    row = hkv * d * 2
    total_blocks = pool_bytes // (2 * L * block_size * row)
    k_pools = [torch.zeros(total_blocks, block_size, hkv, d, device=dev, dtype=torch.bfloat16) for _ in range(L)]
    v_pools = [torch.zeros_like(k_pools[0]) for _ in range(L)]
    pool = _BlockPool(total_blocks, block_size)
    max_blocks = -(-g.max_context // block_size)
    max_prompt = max((p for _, p, _ in records), default=1)
    gen = torch.Generator(device=dev).manual_seed(0)
    q_pf = torch.randn(max_prompt, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    k_pf = torch.randn(1, max_prompt, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    v_pf = torch.randn_like(k_pf)
    q_dec = torch.randn(g.max_batch, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    k_dec = torch.randn(g.max_batch, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    v_dec = torch.randn_like(k_dec)
    out_pf, out_dec = torch.empty_like(q_pf), torch.empty_like(q_dec)
    table_host = torch.zeros(g.max_batch, max_blocks, dtype=torch.int32).pin_memory()
    table_dev = torch.zeros(g.max_batch, max_blocks, dtype=torch.int32, device=dev)
    seq_host = torch.zeros(g.max_batch, dtype=torch.int32).pin_memory()
    seq_dev = torch.zeros(g.max_batch, dtype=torch.int32, device=dev)
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    token_bytes = 2 * g.n_layers * g.per_token_layer_bytes

    metrics = ServingMetrics()
    pending: deque = deque(enumerate(records))
    running: dict[int, _Running] = {}
    free_slots = deque(range(g.max_batch))
    admit_counter = 0
    iteration = 0
    t_start = time.perf_counter()
    while pending or running:
        t0 = time.perf_counter()
        clock_ms = (t0 - t_start) * 1e3
        if not running and pending and pending[0][1][0] > clock_ms:
            time.sleep((pending[0][1][0] - clock_ms) / 1e3)
            clock_ms = pending[0][1][0]
        t_exp = time.perf_counter()
        while pending and pending[0][1][0] <= clock_ms and free_slots:
            idx, rec = pending.popleft()
            rid = free_slots.popleft()
            running[rid] = _Running(idx, rec[1], rec[2], ctx=rec[1], admit_order=admit_counter)
            admit_counter += 1
            metrics.req_arrival_ms.setdefault(idx, float(rec[0]))
            metrics.req_admit_ms.setdefault(idx, clock_ms)
        preempted = 0
        for rid in sorted(running, key=lambda r: running[r].admit_order):
            while rid in running and not pool.grow(rid, running[rid].ctx):
                victim = max(running, key=lambda r: running[r].admit_order)
                st = running.pop(victim)
                pool.release(victim)
                free_slots.append(victim)
                pending.appendleft((st.record_index, records[st.record_index]))
                preempted += 1
                metrics.preemptions += 1
                if metrics.preemptions > preemption_cap:
                    raise SimulationAborted("paged: preemption cap")
        pf = [rid for rid, r in running.items() if r.produced == 0]
        dec = [rid for rid, r in running.items() if r.produced > 0]
        # host-side block-table preparation for this iteration (padded [B, max_blocks])
        tbl = table_host.numpy()
        sq = seq_host.numpy()
        order = pf + dec
        for i, rid in enumerate(order):
            blks = pool.owned[rid]
            tbl[i, :len(blks)] = blks
            sq[i] = running[rid].ctx - (1 if rid in dec else 0)
        table_dev.copy_(table_host, non_blocking=True)
        seq_dev.copy_(seq_host, non_blocking=True)
        exposed_ms = (time.perf_counter() - t_exp) * 1e3
        t_k = time.perf_counter()
        batch = len(running)
        if batch:
            for i, rid in enumerate(pf):
                n = running[rid].ctx
                for layer in range(L):
                    kv_append_paged(k_pools[layer], v_pools[layer], k_pf[:, :n], v_pf[:, :n],
                                    table_dev[i:i + 1], zero)
                    prefill_attention_paged(q_pf[:n], k_pools[layer], v_pools[layer], table_dev[i], n,
                                            out=out_pf[:n])
            if dec:
                o = len(pf)
                Bd = len(dec)
                tb = table_dev[o:o + Bd]
                before = seq_dev[o:o + Bd]
                after = before + 1
                for layer in range(L):
                    kv_append_paged(k_pools[layer], v_pools[layer], k_dec[:Bd], v_dec[:Bd], tb, before)
                    decode_attention_paged(q_dec[:Bd], k_pools[layer], v_pools[layer], tb, after, out=out_dec[:Bd])
            if dense_proxy is not None:
                tokens_now = sum(running[r].ctx for r in pf) + len(dec)
                if hasattr(dense_proxy, "launch"):
                    dense_proxy.launch(tokens_now)
                else:
                    check(lib().vattn_compute_proxy(int(dense_proxy.compute_ms(tokens_now) * 1e6),
                                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
            torch.cuda.synchronize()
        kernel_ms = (time.perf_counter() - t_k) * 1e3
        tokens = sum(r.ctx for r in running.values())
        metrics.iterations.append(IterationRecord(
            iteration=iteration, end_ms=(time.perf_counter() - t_start) * 1e3, batch=batch, prefills=len(pf),
            tokens=tokens, compute_ms=kernel_ms, sync_alloc_ms=0.0, stall_ms=exposed_ms, cpu_ms=exposed_ms,
            committed_bytes=sum(len(b) for b in pool.owned.values()) * block_size * token_bytes,
            used_bytes=tokens * token_bytes, alloc_bytes=0, preemptions=preempted, exposed_ms=exposed_ms,
            kernel_ms=kernel_ms))
        end_ms = metrics.iterations[-1].end_ms
        for rid in list(running):
            st = running[rid]
            if st.produced == 0:
                metrics.req_first_token_ms.setdefault(st.record_index, end_ms)
            st.produced += 1
            if st.produced >= st.decode_tokens:
                metrics.completed_requests += 1
                metrics.generated_tokens += st.decode_tokens
                pool.release(rid)
                del running[rid]
                free_slots.append(rid)
                free_slots = deque(sorted(free_slots))
            else:
                st.ctx += 1
        iteration += 1
    del k_pools, v_pools
    torch.cuda.empty_cache()
    return metrics
