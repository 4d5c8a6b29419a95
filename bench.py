"""Benchmark of the vAttention hot path on B200 (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload l8_decode|y34_decode] [--gather none|fused|nccl] [--eager]

Default workload = BASELINE config 2 (Llama-3-8B-shaped decode: 32 layers, 32 Q / 8 KV heads,
D 128, batch 64, context 4K, bf16, 2 MiB pages).  One step = one decode iteration of the whole
KV cache: allocator `step` (+ the background thread mapping the next iteration's pages), then
per layer one fused launch that appends the new token's K/V and runs decode attention over the
row (timed steps replay one CUDA graph each; `--eager` launches them one by one).  `value` is
decode tokens/s with inputs resident in HBM; `e2e` is the same through the public API with the
inputs copied H2D from pinned host memory and the outputs read back D2H every step.  Extras
(N = 1): decode growth across page-groups, Yi-6B prefill, paged-layout comparisons, shard
shapes, flash-attn / cuDNN, and the config-5 serving trace.

Multi-GPU (torchrun, one process per GPU): KV heads are sharded (geometry.with_tp(N)); every
rank runs an independent allocator + kernels over its heads, no data-path collective; the whole
job's tokens/s = B / (max-over-ranks step time).  Total work is fixed -> "strong" scaling.
"""

from __future__ import annotations

import argparse
import json
import re
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MB2 = 2 * 1024 * 1024
GIB = 1024 ** 3


# ----------------------------------------------------------------------------- utilities
def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None
        self._nvml = None          # (pynvml, handle) when NVML is usable
        self._stop = threading.Event()
        self._samples: list[tuple[float, float, int]] = []

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:   # the CUDA device's NVML handle by UUID (CUDA_VISIBLE_DEVICES may renumber)
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.dev).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid)
        except Exception:   # noqa: BLE001
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def _nvml_loop(self):
        nv, h = self._nvml
        smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self._stop.is_set():
            try:
                self._samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), smax,
                                      int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:   # noqa: BLE001
                break
            self._stop.wait(0.005)

    def start(self):
        # NVML in-process every 5 ms (no start-up lag, so short timed regions get many samples);
        # nvidia-smi -lms 100 when NVML is unavailable
        try:
            self._nvml = self._nvml_handle()
            self._t = threading.Thread(target=self._nvml_loop, daemon=True)
            self._t.start()
            return
        except Exception:   # noqa: BLE001
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            nv = self._nvml[0]
            bits = {"hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                    "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                    "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                    "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)}
            sm = [x[0] for x in self._samples]
            reasons = {n for n, b in bits.items() for x in self._samples if x[2] & b}
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self._samples[-1][1] if self._samples else None,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def box_copy_gbs(dev) -> float:
    """HBM copy bandwidth of THIS GPU, measured the way MEASURED_PEAKS.json's hbm_gbs is
    (b.copy_(a) over 1 Gi bf16 elements, read + write bytes, best of 10): B200 boxes of the pool
    differ by ~10 % in HBM throughput, so the line also reports the fraction against this box."""
    import torch

    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * (1 << 30) * 2 / (best * 1e-3) / 1e9


def traffic_lookup(kernel: str, shape: str, algorithmic_bytes: float):
    """ncu DRAM traffic (read + write bytes per launch, one `ncu --set full` capture) of `kernel`
    at the workload shape `shape` from profiles/ncu_traffic.json, scaled to this run's
    algorithmic bytes when the capture's context differs slightly; (None, why) if not captured."""
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if not tf.exists():
        return None, "no profiles/ncu_traffic.json"
    # the capture is of the decode kernel itself: drop the split-merge part of the label
    kernel_key = re.sub(r" \(cluster combine\)| \+ decode_combine_kernel<\d+>", "", kernel)
    ent = json.loads(tf.read_text()).get(f"{kernel_key}|{shape}")
    if not ent:
        return None, f"no ncu capture of {kernel} at {shape}"
    t = ent["traffic_bytes"]
    if ent.get("algorithmic_bytes"):
        t = t * algorithmic_bytes / ent["algorithmic_bytes"]
    return t, f"profiles/ncu_traffic.json[{kernel}|{shape}] ({ent.get('capture', 'ncu --set full')})"


def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("VATTN_BENCH_ONE_GPU"):   # test harness: every rank on cuda:0 (gloo backend)
        local = 0
    if torch.cuda.is_available():
        torch.cuda.set_device(local)             # before NCCL binds its communicator to a device
    if world > 1 and not dist.is_initialized():
        backend = os.environ.get("VATTN_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend=backend)
    return world, rank, local


def _reduce_device():
    import torch
    import torch.distributed as dist

    nccl = dist.is_initialized() and dist.get_backend() == "nccl"
    return torch.device("cuda") if nccl else torch.device("cpu")


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- workloads
def decode_geometry(workload: str, world: int):
    from paper_2405_04437_b200.geometry import llama3_8b, yi_34b

    if workload == "l8_decode":
        g = llama3_8b(max_context=8192, max_batch=64)
        ctx = 4096
        name = "llama-3-8b decode b64 ctx4096 (32 layers)"
    elif workload == "y34_decode":
        # Yi-34B at G=1 does not fit (60 layers x 4 GiB); per-layer throughput on 8 layers
        g = yi_34b(max_context=8448, max_batch=128)
        g = g.__class__(**{**g.to_dict(), "n_layers": 8})
        ctx = 8192
        name = "yi-34b decode b128 ctx8192 (8 of 60 layers timed)"
    else:
        raise ValueError(workload)
    return g.with_tp(world), ctx, name


def bench_decode(args, world, rank, local):
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import (decode_attention, decode_attention_append, decode_attention_gather,
                                                 decode_kernel_name, decode_num_splits, kv_append)
    from paper_2405_04437_b200.parallel import gather_heads

    dev = torch.device("cuda", local)
    g, ctx, wname = decode_geometry(args.workload, world)
    B, N = g.max_batch, g.n_layers
    hkv, hq, d = g.kv_heads_per_worker, g.q_heads_per_worker, g.head_dim
    steps, warm = args.steps, args.warmup
    # pool: every slot at ctx + all the steps this run takes (warm-up, timed, e2e), + slack
    groups = math.ceil((ctx + steps + warm + 1 + max(3, min(steps, 20)) + 4) * g.per_token_layer_bytes / MB2)
    pool = (groups * B + B // 8 + 1) * 2 * N * MB2   # every slot's groups + a little slack (fewer cuMemCreate at init)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=pool, eager_groups=0,
                                          reclaim_threshold=0.0), backend="cuda", device=local)
    t0 = time.perf_counter()
    rids = [mgr.alloc_reqid() for _ in range(B)]
    seq = [0] * B
    for r in rids:
        seq[r] = ctx
    res0 = mgr.step(seq)
    assert res0.ok
    prefill_map_s = time.perf_counter() - t0
    # synthetic K/V history: fill each layer's cache rows [0, ctx) (prefill-style append)
    gen = torch.Generator(device=dev).manual_seed(0)
    zeros = torch.zeros(B, dtype=torch.int32, device=dev)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    chunk = 512
    for layer in range(N):
        for c0 in range(0, ctx, chunk):
            kn = torch.randn(B, chunk, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
            vn = torch.randn(B, chunk, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
            kv_append(mgr, layer, kn, vn, zeros + c0, idx)
    torch.cuda.synchronize()
    # per-step inputs (resident): q, new k/v per layer
    q = torch.randn(N, B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    kn = torch.randn(N, B, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    vn = torch.randn(N, B, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    out = torch.empty(N, B, hq, d, device=dev, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)     # row the new token goes to
    stream = torch.cuda.current_stream()

    state = {"seq": list(seq), "pos": pos}
    splits = decode_num_splits(B, hkv, ctx + 1)
    hg = None
    if args.gather == "fused" and world > 1:
        from paper_2405_04437_b200.parallel import HeadGather
        hg = HeadGather.create(B, hq * world, d, device=local)

    def launch_layers(dec_events, q_, kn_, vn_, out_, st, pre_layer=None, post_layer=None):
        p = state["pos"]
        for layer in range(N):
            if pre_layer is not None:
                pre_layer(layer)
            timed = dec_events is not None and dec_events[layer] is not None
            if timed:
                dec_events[layer][0].record(st)
            if hg is not None:      # fused decode + head all-gather over peer memory
                decode_attention_gather(mgr, layer, q_[layer], hg, p, idx, k_new=kn_[layer], v_new=vn_[layer],
                                        num_splits=splits)
            elif args.gather == "nccl":
                decode_attention_append(mgr, layer, q_[layer], kn_[layer], vn_[layer], p, idx,
                                        out=out_[layer], num_splits=splits)
                gather_heads(out_[layer])
            elif args.unfused:
                kv_append(mgr, layer, kn_[layer], vn_[layer], p, idx)
                decode_attention(mgr, layer, q_[layer], p + 1, idx, out=out_[layer], num_splits=splits)
            else:   # one launch: append the new token at row p and attend over p + 1 rows
                decode_attention_append(mgr, layer, q_[layer], kn_[layer], vn_[layer], p, idx,
                                        out=out_[layer], num_splits=splits)
            if timed:
                dec_events[layer][1].record(st)
            if post_layer is not None:
                post_layer(layer)

    def one_step(dec_events=None, q_=q, kn_=kn, vn_=vn, out_=out, pre_layer=None, post_layer=None, graph=None):
        nxt = list(state["seq"])
        for r in rids:
            nxt[r] += 1
        t_h = time.perf_counter()
        r = mgr.step(nxt)                       # joins the bg window, maps any shortfall
        exposed = time.perf_counter() - t_h
        assert r.ok
        if graph is not None:
            graph.replay()                      # layers + position update, one host call
        else:
            launch_layers(dec_events, q_, kn_, vn_, out_, stream, pre_layer, post_layer)
            state["pos"].add_(1)
        state["seq"] = nxt
        nn = list(nxt)
        for rr in rids:
            nn[rr] += 1
        mgr.plan_overlap(nn)
        mgr.bg_submit()                         # next iteration's maps run during these kernels
        return exposed

    for _ in range(warm):
        one_step()
    torch.cuda.synchronize()
    use_graph = not args.eager and args.gather != "nccl"   # NCCL stays eager
    if use_graph:
        # One CUDA graph per timed step (the 32 fused append+decode launches, the per-layer
        # timing events as external record nodes, and the row-position update), so the timed
        # step costs one replay on the host.  Captured, not executed: state is unchanged.
        mgr.bg_wait()
        # Timing events inside the graph are record nodes between consecutive decode launches and
        # cancel their programmatic dependent launch (each costs the overlap of a layer's tail
        # with the next layer's K/V streaming), so by default none are captured and a launch's
        # time is its share of the device-timed step (the step is the 32 decode launches and a
        # one-element position update).  VATTN_BENCH_EVENT_STRIDE=k brackets every k-th layer.
        stride = int(os.environ.get("VATTN_BENCH_EVENT_STRIDE", "0"))
        ev = [[(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
               if stride > 0 and layer % stride == 0 else None for layer in range(N)] for _ in range(steps)]
        cap = torch.cuda.Stream(device=dev)
        graphs = []
        for i in range(steps):
            gr = torch.cuda.CUDAGraph()
            cap.wait_stream(stream)
            with torch.cuda.graph(gr, stream=cap, capture_error_mode="thread_local"):
                launch_layers(ev[i], q, kn, vn, out, torch.cuda.current_stream())
                state["pos"].add_(1)
                mgr.mark_use()          # one unmap-fence node closing the captured step
            graphs.append(gr)
        torch.cuda.synchronize()
    else:
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(N)] for _ in range(steps)]
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    exposed = []
    s0.record(stream)
    for i in range(steps):
        exposed.append(one_step(ev[i], graph=graphs[i] if use_graph else None))
    s1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms_total = s0.elapsed_time(s1)
    dec_ms = [a.elapsed_time(b) for row in ev for pair in row if pair is not None for a, b in [pair]]
    ms_step = max_over_ranks(ms_total / steps)
    tokens_s = B / (ms_step / 1e3)
    mean_ctx = ctx + warm + 1 + (steps - 1) / 2
    dec_bytes = 2 * B * mean_ctx * hkv * d * 2 + 2 * B * hq * d * 2     # algorithmic, per launch
    # per-launch time: the bracketed launches when events were captured, else the launch's share
    # of the device-timed step (an upper bound: the step also holds the position update)
    dec_us = statistics.mean(dec_ms) * 1e3 if dec_ms else ms_total / steps / N * 1e3
    dec_timing = "cuda events around launches" if dec_ms else "step / 32 launches (cuda events around the timed steps)"
    pk = peaks()
    achieved = dec_bytes / (dec_us * 1e-6) / 1e9
    box_copy = box_copy_gbs(dev)
    kernel_name = decode_kernel_name(B, hkv, ctx + 1, splits, d) + ("" if args.unfused else " (fused append)")
    traffic, traffic_src = traffic_lookup(kernel_name, f"{args.workload}-G{world}", dec_bytes)

    # ---- e2e through the public API with host buffers (pinned) ----
    qh = q.cpu().pin_memory()
    knh, vnh = kn.cpu().pin_memory(), vn.cpu().pin_memory()
    outh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    q_d, kn_d, vn_d = torch.empty_like(q), torch.empty_like(kn), torch.empty_like(vn)
    e2e_steps = max(3, min(steps, 20))

    # Per-layer pipelined transfers: layer l's q/k/v H2D (one copy stream) and its output D2H
    # (a second stream, PCIe is full duplex) overlap the kernels of the neighbouring layers.
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    h2d_ev = [torch.cuda.Event() for _ in range(N)]
    done_ev = [torch.cuda.Event() for _ in range(N)]
    first = [True]

    def pre_layer(layer):
        stream.wait_event(h2d_ev[layer])

    def post_layer(layer):
        done_ev[layer].record(stream)
        d2h_s.wait_event(done_ev[layer])
        with torch.cuda.stream(d2h_s):
            outh[layer].copy_(out[layer], non_blocking=True)

    def e2e_step():
        h2d_s.wait_stream(stream)
        with torch.cuda.stream(h2d_s):
            for layer in range(N):
                if not first[0]:
                    h2d_s.wait_event(done_ev[layer])     # previous step finished reading layer l
                q_d[layer].copy_(qh[layer], non_blocking=True)
                kn_d[layer].copy_(knh[layer], non_blocking=True)
                vn_d[layer].copy_(vnh[layer], non_blocking=True)
                h2d_ev[layer].record(h2d_s)
        first[0] = False
        one_step(None, q_d, kn_d, vn_d, out, pre_layer=pre_layer, post_layer=post_layer)
        stream.wait_stream(d2h_s)                       # the step ends when its outputs are on the host

    if use_graph:
        # Graph path: the copies are pipelined ACROSS steps instead of per layer (a per-layer
        # event wait between two decode launches cancels their programmatic dependent launch):
        # step i's q/k/v land in buffer set i % 2 while step i - 1 computes, and step i's outputs
        # go to the host while step i + 1 computes.  Every step still moves its own inputs H2D
        # and its outputs D2H inside the timed region.
        qb, knb, vnb, ob = ([torch.empty_like(t) for _ in range(2)] for t in (q, kn, vn, out))
        gr2 = []
        for par in range(2):
            g2 = torch.cuda.CUDAGraph()
            cap.wait_stream(stream)
            with torch.cuda.graph(g2, stream=cap, capture_error_mode="thread_local"):
                launch_layers(None, qb[par], knb[par], vnb[par], ob[par], torch.cuda.current_stream())
                state["pos"].add_(1)
                mgr.mark_use()
            gr2.append(g2)
        torch.cuda.synchronize()
        in_ev = [torch.cuda.Event() for _ in range(2)]
        comp_ev = [torch.cuda.Event() for _ in range(2)]
        out_ev = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]

        def h2d(par):
            if used[par]:
                h2d_s.wait_event(comp_ev[par])          # step i - 2 finished reading buffer set par
            with torch.cuda.stream(h2d_s):
                qb[par].copy_(qh, non_blocking=True)
                knb[par].copy_(knh, non_blocking=True)
                vnb[par].copy_(vnh, non_blocking=True)
            in_ev[par].record(h2d_s)

        def run_e2e(n_steps):
            h2d(0)
            for i in range(n_steps):
                par = i % 2
                if i + 1 < n_steps:
                    h2d(1 - par)
                stream.wait_event(in_ev[par])
                if used[par]:
                    stream.wait_event(out_ev[par])       # step i - 2's outputs left buffer par
                one_step(None, graph=gr2[par])
                comp_ev[par].record(stream)
                used[par] = True
                d2h_s.wait_event(comp_ev[par])
                with torch.cuda.stream(d2h_s):
                    outh.copy_(ob[par], non_blocking=True)
                out_ev[par].record(d2h_s)
            stream.wait_stream(d2h_s)

        run_e2e(2)
        torch.cuda.synchronize()
        barrier()
        used[0] = used[1] = False
        s0.record(stream)
        run_e2e(e2e_steps)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / e2e_steps)
        e2e_pipeline = "inputs of step i+1 H2D and outputs of step i-1 D2H under step i's compute (graph replay per step)"
    else:
        e2e_step()
        torch.cuda.synchronize()
        barrier()
        s0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / e2e_steps)
        e2e_pipeline = "per-layer H2D / D2H overlapping neighbouring layers (eager launches)"
    h2d_bytes = qh.numel() * 2 + knh.numel() * 2 + vnh.numel() * 2
    d2h_bytes = outh.numel() * 2
    gather_cmp = None
    if world > 1:
        try:   # a diagnostic: it must not void the headline line
            gather_cmp = head_gather_compare(mgr, q, out, pos, idx, splits, world, local)
        except Exception as e:
            gather_cmp = {"error": repr(e)[:300]}
    st = mgr.driver_stats()
    result = {
        "metric": "decode_attn_tokens_per_s",
        "value": tokens_s * 1.0,
        "unit": "tokens/s",
        "ms_per_step": ms_step,
        "workload": wname,
        "geometry": {"n_layers": N, "batch": B, "context": ctx, "hq": hq, "hkv": hkv, "d": d,
                     "page_group": MB2},
        "decode_kernel_us_mean": dec_us,
        "decode_num_splits": splits,
        "decode_launches_timed": len(dec_ms) if dec_ms else steps * N,
        "decode_kernel_timing": dec_timing,
        "decode_hbm_gbs": achieved,
        "decode_bytes_per_launch": dec_bytes,
        "exposed_map_ms_per_iter": statistics.mean(exposed) * 1e3,
        "exposed_map_ms_max": max(exposed) * 1e3,
        "prefill_map_ms": prefill_map_s * 1e3,
        "driver": {k: st[k] for k in ("real_maps", "real_set_access_calls", "real_map_wall_us",
                                      "real_set_access_wall_us", "real_creates", "init_wall_us")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "copy_peak_this_box_gbs": box_copy, "frac_of_this_box_copy_peak": achieved / box_copy,
                     "algorithmic_bytes": dec_bytes, "kernel": kernel_name,
                     "peak_source": pk["source"], "traffic_source": traffic_src},
        "e2e": {"value": B / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "ms_per_step": e2e_ms, "pipeline": e2e_pipeline},
        "clocks": clk,
        "gpu_launches": steps * N * ((2 if args.unfused and hg is None else 1) + (1 if splits > 8 else 0)
                                     + (1 if hg is not None else 0)),
        "head_gather_mode": args.gather if world > 1 else "none (1 GPU)",
        "decode_kernel_mode": "unfused append+decode" if args.unfused else "fused append+decode (k=/v= semantics)",
    }
    if gather_cmp is not None:
        result["head_gather"] = gather_cmp
    if hg is not None:
        hg.close()
    mgr.close()
    return result


def head_gather_compare(mgr, q, out, pos, idx, splits, world, local, iters=20):
    """N>1 only (all ranks): one layer's decode alone, with the fused peer-memory head gather,
    and followed by an NCCL all_gather of the heads; device time, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2405_04437_b200.attention import decode_attention, decode_attention_gather
    from paper_2405_04437_b200.parallel import HeadGather, gather_heads

    B, hq, d = q.shape[1], q.shape[2], q.shape[3]
    stream = torch.cuda.current_stream()
    hg, err = None, None
    try:
        hg = HeadGather.create(B, hq * world, d, device=local)
    except Exception as e:          # report, but every rank must agree before timing
        err = repr(e)[:200]
    ok = torch.tensor([0 if err else 1], device=_reduce_device())
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / iters * 1e3)

    res = {"layer_decode_us": timed(lambda: decode_attention(mgr, 0, q[0], pos, idx, out=out[0], num_splits=splits))}
    nccl = dist.get_backend() == "nccl"
    if nccl:
        res["nccl_us"] = timed(lambda: gather_heads(decode_attention(mgr, 0, q[0], pos, idx, out=out[0],
                                                                     num_splits=splits)))
    if int(ok.item()) == 1:
        res["fused_us"] = timed(lambda: decode_attention_gather(mgr, 0, q[0], hg, pos, idx, num_splits=splits))
        got = decode_attention_gather(mgr, 0, q[0], hg, pos, idx, num_splits=splits)
        mine = decode_attention(mgr, 0, q[0], pos, idx, out=out[0], num_splits=splits)
        torch.cuda.synchronize()
        r0 = dist.get_rank() * hq
        res["fused_rows_equal_local"] = bool(torch.equal(got[:, r0:r0 + hq], mine))
        if nccl:
            res["fused_equals_nccl"] = bool(torch.equal(gather_heads(mine), got))
        res["timed_out_ranks"] = hg.timed_out_ranks()
    else:
        res["fused_error"] = err or "a peer rank failed to set up the gather"
    if hg is not None:
        hg.close()
    res["bytes_per_rank"] = B * hq * d * 2
    return res


# ----------------------------------------------------------------------------- extras
def _time_ms(fn, iters=10, warm=3):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def extra_prefill(local):
    """BASELINE config 3: Yi-6B 16K prompt appended into a request slot of the virtual cache,
    then causal tcgen05 prefill attention over it (one layer; 32 Q / 4 KV heads, D 128)."""
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import kv_append, prefill_attention
    from paper_2405_04437_b200.geometry import yi_6b

    dev = torch.device("cuda", local)
    S = 16384
    g = yi_6b(max_context=S, max_batch=1)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2), device=local)
    rid = mgr.alloc_reqid()
    t0 = time.perf_counter()
    assert mgr.step([S]).ok
    map_ms = (time.perf_counter() - t0) * 1e3
    gen = torch.Generator(device=dev).manual_seed(0)
    kn = torch.randn(1, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    vn = torch.randn(1, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    q = torch.randn(S, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    idx = torch.tensor([rid], dtype=torch.int32, device=dev)
    app_ms = _time_ms(lambda: kv_append(mgr, 0, kn, vn, zero, idx), iters=20)
    pf_ms = _time_ms(lambda: prefill_attention(mgr, 0, q, rid, out=out), iters=10)
    pk = peaks()
    flops = 2.0 * S * S * 128 * 32
    tf = flops / (pf_ms * 1e-3) / 1e12
    app_bytes = 2 * 2 * S * 4 * 128 * 2
    # paged-layout variant of the same kernel on identical K/V (PAPER.md:606-623 comparison)
    from paper_2405_04437_b200.attention import prefill_attention_paged
    paged = {}
    kc, vc = mgr.k_cache(0)[rid, :S].contiguous(), mgr.v_cache(0)[rid, :S].contiguous()
    for bs in (16, 256):
        nb = S // bs
        perm = torch.randperm(nb, device=dev, generator=gen)
        kp = torch.empty(nb, bs, 4, 128, device=dev, dtype=torch.bfloat16)
        vp = torch.empty_like(kp)
        kp[perm] = kc.view(nb, bs, 4, 128)
        vp[perm] = vc.view(nb, bs, 4, 128)
        bt = perm.to(torch.int32)
        ms = _time_ms(lambda: prefill_attention_paged(q, kp, vp, bt, S), iters=10)
        paged[f"paged_bs{bs}_ms"] = ms
        paged[f"paged_bs{bs}_slowdown"] = ms / pf_ms
    mgr.close()
    return {"workload": "yi-6b prefill 16K causal (1 layer, 32 Q / 4 KV heads, D 128)",
            "prefill_ms": pf_ms, "prefill_tflops": tf,
            "prefill_frac_of_measured_burst": tf / pk["bf16_tflops"], "prefill_frac_of_2250_nominal": tf / 2250.0,
            "flops": flops, "append_us": app_ms * 1e3, "append_gbs": app_bytes / (app_ms * 1e-3) / 1e9,
            "append_frac_hbm": app_bytes / (app_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
            "map_16k_prompt_ms": map_ms, **paged}


def bench_prefill(local, iters=10, cpu=True):
    """BASELINE config 3 as a measured contract object (top-level `prefill` of the bench line):
    Yi-6B-shaped 16K-token prompt (32 Q / 4 KV heads, D 128, one layer, causal) appended into a
    request slot of the virtual cache, then the tcgen05 prefill kernel over it.

    * value / roofline: prefill kernel TFLOP/s (causal flops 2*S^2*D*Hq, the FlashAttention
      convention) by CUDA events around each launch, against the measured dense bf16 burst peak
      (the kernel is timed alone); q/out are 128 MiB each, larger than L2.
    * append: KV append of 4 requests x 16K tokens in one launch (134 MiB read + 134 MiB written,
      above the 126 MB L2), L2 flushed by a 256 MiB write before each timed launch.
    * e2e: the public API from pinned host buffers: q/k/v H2D, kv_append, prefill, output D2H.
    * cpu_baseline: the fp32 oracle restatement (oracle/attention.py prefill_ref) on all host
      cores over 8 of the 32 query heads (one KV head's GQA group, all 16K rows), scaled x4."""
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import kv_append, prefill_attention
    from paper_2405_04437_b200.geometry import yi_6b

    dev = torch.device("cuda", local)
    S, R = 16384, 4
    hq, hkv, d = 32, 4, 128
    g = yi_6b(max_context=S, max_batch=R)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * R * 8 + 4) * MB2), device=local)
    rids = [mgr.alloc_reqid() for _ in range(R)]
    t0 = time.perf_counter()
    assert mgr.step([S] * R).ok
    map_ms = (time.perf_counter() - t0) * 1e3
    gen = torch.Generator(device=dev).manual_seed(0)
    kn = torch.randn(R, S, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    vn = torch.randn(R, S, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    q = torch.randn(S, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    zeros = torch.zeros(R, dtype=torch.int32, device=dev)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    # L2 flush by READING 256 MiB (a write would leave ~126 MB of dirty lines whose write-back
    # would be charged to the timed launch)
    flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()

    def per_launch(fn, n, flush_l2):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            if flush_l2:
                flush.amax()
            e0.record(st)
            fn()
            e1.record(st)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    app_ms = per_launch(lambda: kv_append(mgr, 0, kn, vn, zeros, idx), iters, True)
    app_bytes = 2 * (2 * R * S * hkv * d * 2)                     # K and V: read source + write cache
    clocks = ClockSampler(local)          # the prefill is tensor-bound: its SM clock is the context
    clocks.start()
    pf_ms = per_launch(lambda: prefill_attention(mgr, 0, q, rids[0], out=out), iters, False)
    clk = clocks.stop()
    pf_mean = statistics.mean(pf_ms)
    flops = 2.0 * S * S * d * hq
    pk = peaks()
    tf = flops / (pf_mean * 1e-3) / 1e12
    traffic, traffic_src = traffic_lookup("prefill_kernel<0,false,128,false>", "y6-16k", flops)
    # e2e through the public API with host buffers
    qh, kh, vh = q.cpu().pin_memory(), kn[:1].cpu().pin_memory(), vn[:1].cpu().pin_memory()
    oh = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    q_d, k_d, v_d = torch.empty_like(q), torch.empty_like(kn[:1]), torch.empty_like(vn[:1])
    one = idx[:1]

    def e2e_once():
        q_d.copy_(qh, non_blocking=True)
        k_d.copy_(kh, non_blocking=True)
        v_d.copy_(vh, non_blocking=True)
        kv_append(mgr, 0, k_d, v_d, zeros[:1], one)
        prefill_attention(mgr, 0, q_d, rids[0], out=out)
        oh.copy_(out, non_blocking=True)

    e2e_serial_ms = statistics.mean(per_launch(e2e_once, max(3, iters // 2), False))
    # Pipelined across prompts (two copy streams, double-buffered device buffers): prompt i + 1's
    # q/k/v go H2D and prompt i - 1's output D2H while prompt i is appended and attended; every
    # prompt still moves all its bytes inside the timed region.
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    qb = [torch.empty_like(q) for _ in range(2)]
    kb = [torch.empty_like(kn[:1]) for _ in range(2)]
    vb = [torch.empty_like(vn[:1]) for _ in range(2)]
    ob = [torch.empty_like(out) for _ in range(2)]
    in_ev = [torch.cuda.Event() for _ in range(2)]
    comp_ev = [torch.cuda.Event() for _ in range(2)]
    out_ev = [torch.cuda.Event() for _ in range(2)]

    def run_pipelined(n):
        used = [False, False]

        def h2d(par):
            if used[par]:
                h2d_s.wait_event(comp_ev[par])
            with torch.cuda.stream(h2d_s):
                qb[par].copy_(qh, non_blocking=True)
                kb[par].copy_(kh, non_blocking=True)
                vb[par].copy_(vh, non_blocking=True)
            in_ev[par].record(h2d_s)

        h2d(0)
        for i in range(n):
            par = i % 2
            if i + 1 < n:
                h2d(1 - par)
            st.wait_event(in_ev[par])
            if used[par]:
                st.wait_event(out_ev[par])
            kv_append(mgr, 0, kb[par], vb[par], zeros[:1], one)
            prefill_attention(mgr, 0, qb[par], rids[0], out=ob[par])
            comp_ev[par].record(st)
            used[par] = True
            d2h_s.wait_event(comp_ev[par])
            with torch.cuda.stream(d2h_s):
                oh.copy_(ob[par], non_blocking=True)
            out_ev[par].record(d2h_s)
        st.wait_stream(d2h_s)

    run_pipelined(2)
    torch.cuda.synchronize()
    n_e2e = max(4, iters // 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run_pipelined(n_e2e)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / n_e2e
    res = {
        "metric": "prefill_attn_tflops", "value": tf, "unit": "TFLOP/s", "dtype": "bf16",
        "workload": "yi-6b prefill, 16K-token prompt, causal, 1 layer (32 Q / 4 KV heads, D 128), 2 MiB pages",
        "ms_per_launch": pf_mean, "launches_timed": len(pf_ms), "flops_per_launch": flops,
        "roofline": {"bound": "tensor", "achieved": tf, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": tf / pk["bf16_tflops"], "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "pf::prefill_kernel<0,false,128,false> (tcgen05.mma cta_group::1, TMEM accumulators)",
                     "peak_source": pk["source"] + " bf16 burst (kernel timed alone)",
                     "frac_of_2250_nominal": tf / 2250.0},
        "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": (qh.numel() + kh.numel() + vh.numel()) * 2,
                "d2h_bytes_per_step": oh.numel() * 2, "ms_per_step": e2e_ms,
                "note": "pinned host q/k/v -> H2D, kv_append, prefill, out -> D2H per prompt, pipelined "
                        "across prompts on two copy streams (PCIe-bound)",
                "serial_ms_per_step": e2e_serial_ms},
        "append": {"workload": f"{R} requests x {S} tokens in one launch (K+V {app_bytes / 2**20:.0f} MiB moved, > L2)",
                   "us_per_launch": statistics.mean(app_ms) * 1e3, "bytes_per_launch": app_bytes,
                   "gbs": app_bytes / (statistics.mean(app_ms) * 1e-3) / 1e9,
                   "frac_hbm": app_bytes / (statistics.mean(app_ms) * 1e-3) / 1e9 / pk["hbm_gbs"],
                   "l2": "256 MiB read (L2 flush, no dirty lines) before every timed launch"},
        "map_16k_prompt_x4_ms": map_ms,
        "gpu_launches": len(pf_ms),
        "clocks": clk,
    }
    if cpu:
        res["cpu_baseline"] = cpu_prefill_baseline(S, hq, hkv, d)
    del kn, vn, flush
    mgr.close()
    torch.cuda.empty_cache()
    return res


def cpu_prefill_baseline(S, hq, hkv, d, head_groups=1):
    """fp32 CPU causal prefill (oracle/attention.py prefill_ref) on all host cores: `head_groups`
    of the hkv GQA groups (all S query rows of those hq/hkv heads), scaled to every head."""
    import torch

    from oracle.attention import prefill_ref

    torch.set_num_threads(host_cores())
    gen = torch.Generator().manual_seed(0)
    grp = hq // hkv
    q = torch.randn(S, grp * head_groups, d, generator=gen).to(torch.bfloat16)
    k = torch.randn(S, head_groups, d, generator=gen).to(torch.bfloat16)
    v = torch.randn(S, head_groups, d, generator=gen).to(torch.bfloat16)
    t0 = time.perf_counter()
    prefill_ref(q, k, v, causal=True)
    dt = (time.perf_counter() - t0) * (hkv / head_groups)
    flops = 2.0 * S * S * d * hq
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": host_cores(), "kind": "port",
            "sample": (f"{head_groups} of {hkv} KV-head groups ({grp * head_groups} of {hq} query heads, all {S} rows, "
                       f"causal) of one layer, fp32 torch restatement oracle/attention.py prefill_ref on "
                       f"{host_cores()} threads, scaled x{hkv / head_groups:g}; cpu: {cpu_model()}"),
            "ms_per_layer": dt * 1e3}


def extra_long_prefill(local, lengths=(4096, 16384, 65536, 131072)):
    """Prefill at growing context (the paper's prefill-throughput figure, PAPER.md:549, 653-660:
    attention dominates from 16K up, where the non-paged kernel's advantage shows): Yi-6B heads
    (32 Q / 4 KV, D 128), causal, one layer, the tcgen05 kernel on a contiguous slot vs the same
    kernel gathering K/V through a block table (blocks of 16 and 256)."""
    import torch

    from paper_2405_04437_b200.attention import prefill_attention_paged, prefill_attention_raw

    dev = torch.device("cuda", local)
    out = {}
    for S in lengths:
        gen = torch.Generator(device=dev).manual_seed(S)
        k = torch.randn(1, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        q = torch.randn(S, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        o = torch.empty_like(q)
        it = 10 if S <= 16384 else 3
        ms = _time_ms(lambda: prefill_attention_raw(q, k, v, 0, S, out=o), iters=it, warm=2)
        flops = 2.0 * S * S * 128 * 32
        row = {"ms": ms, "tflops": flops / (ms * 1e-3) / 1e12}
        for bs in (16, 256):
            nb = S // bs
            perm = torch.randperm(nb, device=dev, generator=gen)
            kp = torch.empty(nb, bs, 4, 128, device=dev, dtype=torch.bfloat16)
            vp = torch.empty_like(kp)
            kp[perm] = k[0].view(nb, bs, 4, 128)
            vp[perm] = v[0].view(nb, bs, 4, 128)
            bt = perm.to(torch.int32)
            pms = _time_ms(lambda: prefill_attention_paged(q, kp, vp, bt, S, out=o), iters=it, warm=2)
            row[f"paged_bs{bs}_slowdown"] = pms / ms
            del kp, vp
        out[f"S{S}"] = row
        del k, v, q, o
        torch.cuda.empty_cache()
    return out


def extra_paged(local):
    """Contiguous (vAttention) vs paged-layout decode kernel on identical K/V (L8 layer)."""
    import torch

    from paper_2405_04437_b200.attention import decode_attention_paged, decode_attention_raw

    dev = torch.device("cuda", local)
    B, hq, hkv, d, L = 64, 32, 8, 128, 4096
    gen = torch.Generator(device=dev).manual_seed(1)
    k = torch.randn(B, L, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    v = torch.randn(B, L, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    q = torch.randn(B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * hkv * d * 2
    res = {"contiguous_us": _time_ms(lambda: decode_attention_raw(q, k, v, seq)) * 1e3}
    for bs in (16, 256):
        nb = L // bs
        perm = torch.randperm(B * nb, device=dev, generator=gen)
        kp = torch.empty_like(k).view(B * nb, bs, hkv, d)
        vp = torch.empty_like(v).view(B * nb, bs, hkv, d)
        kp[perm] = k.view(B * nb, bs, hkv, d)
        vp[perm] = v.view(B * nb, bs, hkv, d)
        bt = perm.view(B, nb).to(torch.int32)
        res[f"paged_bs{bs}_us"] = _time_ms(lambda: decode_attention_paged(q, kp, vp, bt, seq)) * 1e3
        o_ref = decode_attention_raw(q, k, v, seq)
        o_pg = decode_attention_paged(q, kp, vp, bt, seq)
        res[f"paged_bs{bs}_max_abs_diff_vs_contiguous"] = float((o_ref.float() - o_pg.float()).abs().max())
        del kp, vp
    for key in list(res):
        if key.endswith("_us"):
            res[key.replace("_us", "_gbs")] = byt / (res[key] * 1e-6) / 1e9
    res["paged_bs16_slowdown"] = res["paged_bs16_us"] / res["contiguous_us"]
    res["paged_bs256_slowdown"] = res["paged_bs256_us"] / res["contiguous_us"]
    return res


def extra_varlen_prefill(local, cases=((16, 512), (8, 2048), (4, 3072))):
    """Several prompts' prefill attention (Llama-3-8B heads, causal, one layer): one launch per
    request vs one varlen launch for all of them (short prompts alone leave most SMs idle)."""
    import torch

    from paper_2405_04437_b200.attention import prefill_attention_raw, prefill_attention_varlen_raw

    dev = torch.device("cuda", local)
    out = {}
    for n_req, S in cases:
        gen = torch.Generator(device=dev).manual_seed(n_req * S)
        k = torch.randn(n_req, S, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        q = torch.randn(n_req * S, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        o = torch.empty_like(q)
        qs = [q[i * S:(i + 1) * S] for i in range(n_req)]
        os_ = [o[i * S:(i + 1) * S] for i in range(n_req)]

        def per_request():
            for i in range(n_req):
                prefill_attention_raw(qs[i], k, v, i, S, out=os_[i])

        t_each = _time_ms(per_request, iters=10)
        t_var = _time_ms(lambda: prefill_attention_varlen_raw(q, k, v, [S] * n_req, list(range(n_req)), out=o),
                         iters=10)
        flops = n_req * 2.0 * S * S * 128 * 32
        out[f"{n_req}x{S}"] = {"per_request_ms": t_each, "varlen_ms": t_var, "speedup": t_each / t_var,
                               "varlen_tflops": flops / (t_var * 1e-3) / 1e12}
        del k, v, q, o
    return out


def extra_long_decode(local, cases=((1, 32768), (1, 131072), (8, 32768), (8, 131072), (16, 65536))):
    """Decode at long contexts (the paper's decode-attention latency table):
    Llama-3-8B heads (32 Q / 8 KV, D 128), batch B x context L, contiguous split-K kernel vs the
    same kernel through a block table (16 / 256).  Four cache copies are cycled so every launch
    reads HBM.  Latency in µs and HBM GB/s."""
    import torch

    from paper_2405_04437_b200.attention import decode_attention_paged, decode_attention_raw, decode_num_splits

    dev = torch.device("cuda", local)
    hq, hkv, d = 32, 8, 128
    out = {}
    for B, L in cases:
        gen = torch.Generator(device=dev).manual_seed(B * 7 + L)
        ncopy = 2 if B * L >= 8 * 131072 else 4
        kv = [(torch.randn(B, L, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16),
               torch.randn(B, L, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)) for _ in range(ncopy)]
        q = torch.randn(B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
        seq = torch.full((B,), L, dtype=torch.int32, device=dev)
        byt = 2 * B * L * hkv * d * 2
        cnt = [0]

        def contiguous():
            k, v = kv[cnt[0] % ncopy]
            cnt[0] += 1
            decode_attention_raw(q, k, v, seq)

        us = _time_ms(contiguous, iters=8) * 1e3
        row = {"us": us, "gbs": byt / (us * 1e-6) / 1e9, "num_splits": decode_num_splits(B, hkv, L)}
        # the same launches replayed from a CUDA graph (one call per cache copy): device time per
        # call without the ~17 us host enqueue that paces the eager loop at small B
        torch.cuda.synchronize()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cap, capture_error_mode="thread_local"):
            for i in range(ncopy):
                k, v = kv[i]
                decode_attention_raw(q, k, v, seq)
        gus = _time_ms(gr.replay, iters=8) * 1e3 / ncopy
        del gr
        row["us_graph"] = gus
        row["gbs_graph"] = byt / (gus * 1e-6) / 1e9
        for bs in (16, 256):
            nb = L // bs
            perm = torch.randperm(B * nb, device=dev, generator=gen)
            k, v = kv[0]
            kp = torch.empty_like(k).view(B * nb, bs, hkv, d)
            vp = torch.empty_like(v).view(B * nb, bs, hkv, d)
            kp[perm] = k.view(B * nb, bs, hkv, d)
            vp[perm] = v.view(B * nb, bs, hkv, d)
            bt = perm.view(B, nb).to(torch.int32)
            pus = _time_ms(lambda: decode_attention_paged(q, kp, vp, bt, seq), iters=8) * 1e3
            row[f"paged_bs{bs}_slowdown"] = pus / us
            del kp, vp
        out[f"B{B}_L{L}"] = row
        del kv
        torch.cuda.empty_cache()
    return out


def extra_libraries(local):
    """Library kernels on identical inputs, for context (not on the product path).
    * flash-attn 2.8.3: the kernels vAttention runs unmodified.
    * cuDNN SDPA through torch.
    Shapes are the L8 decode layer and the Y6 16K causal prefill."""
    import torch

    from paper_2405_04437_b200.attention import decode_attention_raw, prefill_attention_raw

    dev = torch.device("cuda", local)
    res = {}
    gen = torch.Generator(device=dev).manual_seed(3)
    B, hq, hkv, d, L = 64, 32, 8, 128, 4096
    k = torch.randn(B, L, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    q = torch.randn(B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * hkv * d * 2
    ours = _time_ms(lambda: decode_attention_raw(q, k, v, seq)) * 1e3
    res["decode_l8_ours_us"] = ours
    try:
        import flash_attn

        q4 = q.unsqueeze(1)
        fa = _time_ms(lambda: flash_attn.flash_attn_with_kvcache(q4, k, v, cache_seqlens=seq)) * 1e3
        res["decode_l8_flash_attn_us"] = fa
        res["decode_l8_flash_attn_gbs"] = byt / (fa * 1e-6) / 1e9
        res["decode_l8_speedup_vs_flash_attn"] = fa / ours
    except Exception as e:
        res["flash_attn_decode_error"] = repr(e)[:200]
    del k, v
    S, hq, hkv = 16384, 32, 4
    kc = torch.randn(1, S, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    vc = torch.randn_like(kc)
    qp = torch.randn(S, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    flops = 2.0 * S * S * d * hq
    ours = _time_ms(lambda: prefill_attention_raw(qp, kc, vc, 0, S))
    res["prefill_y6_ours_tflops"] = flops / (ours * 1e-3) / 1e12
    try:
        import flash_attn

        fa = _time_ms(lambda: flash_attn.flash_attn_func(qp.unsqueeze(0), kc, vc, causal=True), iters=5)
        res["prefill_y6_flash_attn_tflops"] = flops / (fa * 1e-3) / 1e12
        res["prefill_y6_speedup_vs_flash_attn"] = fa / ours
    except Exception as e:
        res["flash_attn_prefill_error"] = repr(e)[:200]
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        qh = qp.transpose(0, 1).unsqueeze(0)                              # [1, Hq, S, D]
        kh = kc[0].repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0)
        vh = vc[0].repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0)
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            cd = _time_ms(lambda: torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True),
                          iters=5)
        res["prefill_y6_cudnn_sdpa_tflops"] = flops / (cd * 1e-3) / 1e12
        res["prefill_y6_speedup_vs_cudnn_sdpa"] = cd / ours
    except Exception as e:
        res["cudnn_prefill_error"] = repr(e)[:200]
    return res


def extra_y34_shards(local):
    """BASELINE config 4 per rank: Yi-34B decode (B 128, ctx 8K, 56 Q / 8 KV heads) with KV heads
    sharded over G GPUs — each rank's shard measured on this GPU (no collective on the path, so
    G ranks run these in parallel; the optional output all-gather is excluded)."""
    import torch

    from paper_2405_04437_b200.attention import decode_attention_append_raw

    dev = torch.device("cuda", local)
    B, L = 128, 8192
    pk = peaks()
    out = {}
    for G in (1, 2, 4, 8):
        hq, hkv = 56 // G, 8 // G
        gen = torch.Generator(device=dev).manual_seed(G)
        k = torch.randn(B, L + 64, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        q = torch.randn(B, hq, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kn = torch.randn(B, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        vn = torch.randn_like(kn)
        pos = torch.full((B,), L - 1, dtype=torch.int32, device=dev)
        us = _time_ms(lambda: decode_attention_append_raw(q, k, v, kn, vn, pos), iters=10) * 1e3
        byt = 2 * B * L * hkv * 128 * 2 + 2 * B * hq * 128 * 2
        out[f"G{G}"] = {"hq": hq, "hkv": hkv, "us_per_layer": us, "gbs": byt / (us * 1e-6) / 1e9,
                        "frac_hbm": byt / (us * 1e-6) / 1e9 / pk["hbm_gbs"], "bytes_per_gpu": byt,
                        "job_tokens_per_s_per_layer": B / (us * 1e-6)}
        del k, v
    return out


def extra_l8_shards(local, steps=20):
    """The headline workload's per-rank step at the KV-head shard shapes of a G = 1/2/4/8 job,
    each run on this GPU: manager + 32 fused append+decode launches replayed from one CUDA graph
    per step (as in the timed region).  Ranks share nothing on this path, so the job's tokens/s
    at G GPUs is B / (per-rank step time); this is the single-GPU prediction the torchrun
    scaling run (N = 2/4/8) checks."""
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append
    from paper_2405_04437_b200.geometry import llama3_8b

    dev = torch.device("cuda", local)
    out = {}
    base = None
    for G in (1, 2, 4, 8):
        g = llama3_8b(max_context=8192, max_batch=64).with_tp(G)
        B, N, hq, hkv, d = g.max_batch, g.n_layers, g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim
        groups = math.ceil((4096 + steps + 8) * g.per_token_layer_bytes / MB2)
        mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(groups + 1) * 2 * N * B * MB2,
                                              eager_groups=0, reclaim_threshold=0.0), backend="cuda", device=local)
        rids = [mgr.alloc_reqid() for _ in range(B)]
        assert mgr.step([4096 + steps + 4] * B).ok
        gen = torch.Generator(device=dev).manual_seed(G)
        q = torch.randn(N, B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
        kn = torch.randn(N, B, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
        o = torch.empty_like(q)
        idx = torch.tensor(rids, dtype=torch.int32, device=dev)
        pos = torch.full((B,), 4096, dtype=torch.int32, device=dev)

        def body():
            for layer in range(N):
                decode_attention_append(mgr, layer, q[layer], kn[layer], kn[layer], pos, idx, out=o[layer])

        body()
        torch.cuda.synchronize()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cap, capture_error_mode="thread_local"):
            body()
            mgr.mark_use()              # one unmap-fence node closing the captured step
        ms = _time_ms(gr.replay, iters=steps)
        del gr
        mgr.close()
        tok = B / (ms / 1e3)
        base = base or tok
        out[f"G{G}"] = {"hq": hq, "hkv": hkv, "ms_per_step": ms, "job_tokens_per_s": tok,
                        "scaling_efficiency_vs_G1": tok / (base * G)}
    return out


def extra_decode_growth(local, steps=96, warm=8):
    """Exposed map ms/iter (BASELINE metric) while decode contexts GROW across page-group
    boundaries: Llama-3-8B shape, 32 layers, B 64, contexts staggered 1024 + 16*b (mean ~1.5K: half the init maps of 4K)
    so a row crosses a 2 MiB group (64 buffers to map) every ~16 steps.  Each step = allocator
    step + 32 fused append+decode launches + a host sync (the token sampling point of a serving
    loop).  Modes: sync (maps inside step), overlapped (the reference's plan_overlap ->
    execute_plan on the background thread during the kernels), overlapped + physical prefetch
    of decode growth 64 tokens ahead (logical state unchanged)."""
    import torch

    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append
    from paper_2405_04437_b200.geometry import llama3_8b

    dev = torch.device("cuda", local)
    g = llama3_8b(max_context=8192, max_batch=64)
    B, N, hq, hkv, d = g.max_batch, g.n_layers, g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim
    ctx0 = [1024 + 16 * b for b in range(B)]
    gen = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(N, B, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    kn = torch.randn(N, B, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    res = {"workload": "llama-3-8b decode b64, ctx 1024+16*b growing, 32 layers, 2 MiB groups",
           "steps": steps}
    for mode, pf in (("sync", 0), ("overlapped", 0), ("overlapped_prefetch64", 64)):
        tok = g.per_token_layer_bytes
        groups = max(math.ceil((c + steps + warm + 2) * tok / MB2) for c in ctx0)
        mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(groups + 1) * 2 * N * B * MB2,
                                              eager_groups=0, reclaim_threshold=0.0),
                             backend="cuda", device=local, prefetch_tokens=pf)
        rids = [mgr.alloc_reqid() for _ in range(B)]
        seq = [0] * B
        for r, c in zip(rids, ctx0):
            seq[r] = c
        assert mgr.step(seq).ok
        idx = torch.tensor(rids, dtype=torch.int32, device=dev)
        pos = torch.tensor([seq[r] for r in rids], dtype=torch.int32, device=dev)
        exposed, crossings = [], 0
        torch.cuda.synchronize()
        st0 = mgr.driver_stats()
        for it in range(warm + steps):
            nxt = [s + 1 for s in seq]
            crossed = sum(1 for a, b in zip(seq, nxt) if a and -(-a * tok // MB2) != -(-b * tok // MB2))
            t0 = time.perf_counter()
            assert mgr.step(nxt).ok
            dt = time.perf_counter() - t0
            for layer in range(N):
                decode_attention_append(mgr, layer, q[layer], kn[layer], kn[layer], pos, idx, out=out[layer])
            pos.add_(1)
            seq = nxt
            if mode != "sync":
                mgr.bg_submit(mgr.plan_overlap([s + 1 for s in seq]), prefetch=pf > 0)
            torch.cuda.synchronize()
            if it >= warm:
                exposed.append(dt * 1e3)
                crossings += crossed
        if mode != "sync":
            mgr.bg_wait()
        st = mgr.driver_stats()
        mgr.close()
        res[mode] = {"exposed_map_ms_per_iter": statistics.mean(exposed), "exposed_map_ms_p99":
                     sorted(exposed)[int(0.99 * (len(exposed) - 1))], "exposed_map_ms_max": max(exposed),
                     "rows_crossing_a_group": crossings, "driver_maps": st["real_maps"] - st0["real_maps"],
                     "set_access_us_per_call": (st["real_set_access_wall_us"] - st0["real_set_access_wall_us"])
                     / max(1, st["real_set_access_calls"] - st0["real_set_access_calls"])}
    return res


def extra_serving(local, requests=128, out_dir=ROOT / "gpurun_out" / "serving_bench"):
    """BASELINE config 5: Algorithm-1 loop on the config-5 trace (Llama-3-8B shape), real kernels
    + the dense layers as real bf16 GEMMs sized to the reference IterationModel (serving.GemmDense),
    sync vs overlapped+deferred+eager (+ the B200 prefetch / staged variants) vs the paged layout.
    Per-iteration CSVs and summaries go to gpurun_out/serving_bench/ (Fig. 11/13 analogs); the
    whole 512-request trace runs in tools/serving_trace.py (profiles/r02_serving512/)."""
    from paper_2405_04437_b200.geometry import llama3_8b
    from paper_2405_04437_b200.serving import GemmDense, load_trace_csv, median_prompt_groups, run, run_paged

    rows = load_trace_csv(ROOT / "tests" / "golden" / "trace_config5.csv")[:requests]
    g = llama3_8b(max_context=4096, max_batch=64)
    eager = median_prompt_groups(rows, g, MB2)
    dense = GemmDense(device=local)
    out_dir.mkdir(parents=True, exist_ok=True)
    out = {"trace": f"tests/golden/trace_config5.csv first {requests} requests", "eager_groups": eager,
           "dense": f"bf16 GEMM units of {dense.unit_ms:.3f} ms sized to IterationModel (10 ms + 0.5 us/token)",
           "csv_dir": str(out_dir.relative_to(ROOT))}
    keys = ("iterations", "tokens_per_s", "exposed_map_ms_per_iter", "exposed_map_ms_p99", "exposed_map_ms_max",
            "sync_alloc_ms_total", "stall_ms_total", "preemptions", "ttft_ms_p50", "ttft_ms_p99", "queue_ms_p50",
            "queue_ms_p99", "mean_waste_bytes", "mean_phys_waste_bytes", "peak_phys_bytes")
    # 128 requests: long enough that pool creation and the first admissions do not decide the
    # ratio (48-request runs swung 0.8-1.06x of paged between boxes).  The 2 MiB-handle overlapped
    # loop stays as the reference-design contrast; every variant of DESIGN §5.1-5.2 over the whole
    # 512-request trace is tools/gpu_serving512.sh (profiles/r02_serving512/).
    variants = {
        "overlapped": dict(mode="overlapped"),
        # 8 MiB physical handles behind the 2 MiB bookkeeping (phys_chunk_groups=4): one
        # cuMemMap + cuMemSetAccess per four page-groups of a buffer
        "sync_chunk4": dict(mode="sync", phys_chunk_groups=4),
        "overlapped_chunk4": dict(mode="overlapped", phys_chunk_groups=4),
        # + physical prefetch, speculative eager, lazy unmap and staged admission
        "overlapped_staged_chunk4": dict(mode="overlapped", prefetch_tokens=256, prefetch_slots=4,
                                         prefetch_slot_tokens=3072, lazy_unmap=True, stage_admission=True,
                                         stage_max_iters=32, hold_worker=True, phys_chunk_groups=4),
    }
    for mode, kw in variants.items():
        m = run(rows, g, clock="wall", page_group_size=MB2, pool_bytes=24 * GIB,
                eager_groups=eager if kw["mode"] == "overlapped" else 0, reclaim_threshold=0.10,
                preemption_cap=100_000, dense_proxy=dense, **kw)
        s = m.summary()
        m.write_iterations_csv(out_dir / f"{mode}.csv")
        m.write_summary_json(out_dir / f"{mode}.json")
        its = m.iterations
        dec = [r.exposed_ms for r in its if r.prefills == 0]
        out[mode] = {k: s[k] for k in keys}
        out[mode]["exposed_map_ms_per_decode_iter"] = sum(dec) / max(1, len(dec))
        out[mode]["exposed_map_ms_median"] = statistics.median([r.exposed_ms for r in its]) if its else 0.0
        out[mode]["exposed_breakdown_ms"] = {k: sum(getattr(r, k) for r in its) for k in
                                             ("t_admit_ms", "t_bgwait_ms", "t_step_ms", "t_retire_ms")}
        out[mode]["driver_set_access_ms_total"] = sum(r.drv_set_access_ms for r in its)
        out[mode]["driver_maps_total"] = sum(r.drv_maps for r in its)
        out[mode]["kernel_ms_total"] = s["kernel_ms_total"]
    # Layer-sliced layout (manager.py:93-96): one page-group spans all 32 layers of 32 tokens, so
    # a request's tail wastes 1/N of what the per-layer layout wastes.  Memory
    # is a property of the allocator state alone: all 512 requests on the model clock (shadow
    # backend, the reference's IterationModel), and the staged wall-clock loop in the sliced layout.
    full = load_trace_csv(ROOT / "tests" / "golden" / "trace_config5.csv")
    waste = {}
    for name, sl in (("layered", False), ("sliced", True)):
        mm = run(full, g, clock="model", backend="shadow", mode="overlapped", page_group_size=MB2,
                 pool_bytes=24 * GIB, eager_groups=median_prompt_groups(full, g, MB2, sliced=sl), sliced=sl,
                 reclaim_threshold=0.10, preemption_cap=100_000).summary()
        waste[name] = {"mean_waste_mib": mm["mean_waste_bytes"] / 2 ** 20,
                       "peak_committed_gib": mm["peak_committed_bytes"] / GIB, "iterations": mm["iterations"]}
    waste["waste_ratio_layered_over_sliced"] = waste["layered"]["mean_waste_mib"] / max(1e-9, waste["sliced"]["mean_waste_mib"])
    out["sliced_vs_layered_512_model_clock"] = waste
    # PagedAttention layout with the in-repo paged kernels (block 16), same trace and proxy
    import torch
    torch.cuda.empty_cache()
    m = run_paged(rows, g, block_size=16, pool_bytes=24 * GIB, dense_proxy=dense, device=local)
    s = m.summary()
    m.write_iterations_csv(out_dir / "paged_bs16.csv")
    m.write_summary_json(out_dir / "paged_bs16.json")
    out["paged_bs16"] = {k: s[k] for k in keys + ("kernel_ms_total",) if k in s}
    out["paged_bs16"]["note"] = "exposed = host block allocation + block-table preparation + upload"
    return out


# ----------------------------------------------------------------------------- CPU baseline
class CpuDecodeStep:
    """Oracle port on the host: the fp32 torch restatement of decode attention
    (oracle/attention.py decode_ref_equal: every batch row over its whole context, all query
    heads, on all host cores) for `layers` layers per step + the oracle allocator's `step` for
    the same iteration (1 thread).  Every layer is computed in full; with layers == n_layers the
    step is the whole decode iteration and nothing is extrapolated.  The layers share one K/V
    array (identical shapes; 1 GiB per layer, far above the host LLC, so every layer streams
    from DRAM as distinct layers would)."""

    def __init__(self, workload: str, world: int, layers: int | None = None):
        import torch

        from oracle.allocator import Geometry, OracleManager

        g, ctx, _ = decode_geometry(workload, world)
        self.g, self.ctx = g, ctx
        self.layers = g.n_layers if layers is None else layers
        self.cores = host_cores()
        torch.set_num_threads(self.cores)
        hkv, hq, d, B = g.kv_heads_per_worker, g.q_heads_per_worker, g.head_dim, g.max_batch
        gen = torch.Generator().manual_seed(0)
        self.k = torch.randn(B, ctx + 1, hkv, d, generator=gen, dtype=torch.bfloat16)
        self.v = torch.randn(B, ctx + 1, hkv, d, generator=gen, dtype=torch.bfloat16)
        self.q = torch.randn(self.layers, B, hq, d, generator=gen, dtype=torch.bfloat16)
        og = Geometry(g.n_layers, g.kv_heads_total, g.head_dim, g.bytes_per_elem, g.max_context, B,
                      g.tp_degree)
        pool = (g.max_context * g.per_token_layer_bytes // MB2 + 2) * 2 * g.n_layers * B * MB2
        self.om = OracleManager(og, MB2, pool_bytes=pool)
        self.rids = [self.om.alloc_reqid() for _ in range(B)]
        self.sl = [0] * B
        for r in self.rids:
            self.sl[r] = ctx
        self.om.step(self.sl)

    def step(self) -> float:
        """Seconds for one decode iteration (scaled by n_layers / layers when layers < n_layers)."""
        from oracle.attention import decode_ref_equal

        t0 = time.perf_counter()
        for r in self.rids:
            self.sl[r] = min(self.sl[r] + 1, self.g.max_context)
        self.om.step(self.sl)
        t_alloc = time.perf_counter() - t0
        t0 = time.perf_counter()
        for layer in range(self.layers):
            decode_ref_equal(self.q[layer], self.k, self.v, self.ctx + 1)
        t_layers = time.perf_counter() - t0
        return t_alloc + t_layers * (self.g.n_layers / self.layers)

    def describe(self) -> str:
        g = self.g
        scope = ("every layer, no extrapolation" if self.layers == g.n_layers else
                 f"{self.layers} of {g.n_layers} identical layers computed in full, scaled x{g.n_layers / self.layers:g}")
        return (f"full decode step: {g.max_batch} rows x ctx {self.ctx + 1} x Hq {g.q_heads_per_worker} / "
                f"Hkv {g.kv_heads_per_worker} x D {g.head_dim}, {scope}; fp32 torch restatement "
                f"oracle/attention.py decode_ref_equal on {self.cores} threads + oracle allocator step "
                f"(1 thread); cpu: {cpu_model()}")


def _cpu_layers(workload: str) -> int | None:
    # Llama-3-8B: the whole 32-layer step (~1-3 s on 16 cores); Yi-34B's 8 layers at B 128 x 8K
    # read 4 GiB each: one full layer per step, scaled to the 8 timed layers
    return None if workload == "l8_decode" else 1


def cpu_baseline(workload: str, world: int, steps: int = 2):
    """Main-arm cpu_baseline (rank 0, N = 1): 1 warm-up + `steps` timed full steps (~10 s)."""
    s = CpuDecodeStep(workload, world, _cpu_layers(workload))
    s.step()
    t = statistics.mean(s.step() for _ in range(steps))
    return {"value": s.g.max_batch / t, "unit": "tokens/s", "cores": s.cores, "kind": "port",
            "sample": s.describe() + f"; mean of {steps} steps after 1 warm-up", "ms_per_step": t * 1e3}


def run_reference(args, world, rank):
    """--impl reference: the reference path's CPU implementation on the host cores.  The reference
    (kvsim) is a hardware-free Python simulator with no attention code, so this arm is the oracle
    port (CpuDecodeStep), whose allocator half is pinned bit-exact to the reference itself
    (tests/test_core_parity.py) and whose attention half follows the paper's equation 2."""
    if rank != 0:
        return None
    # the whole job's work (every KV head) on the one host, whatever N is: the host cores do not
    # multiply with the GPU count
    s = CpuDecodeStep(args.workload, 1, _cpu_layers(args.workload))
    for _ in range(args.warmup):
        s.step()
    times = [s.step() for _ in range(args.steps)]
    ms = statistics.mean(times) * 1e3
    _, _, wname = decode_geometry(args.workload, 1)
    val = s.g.max_batch / (ms / 1e3)
    return {
        "impl": "reference", "metric": "decode_attn_tokens_per_s", "value": val, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded randn K/V/Q)",
        "config": {"workload": wname, "parallelism": f"host CPU, full job (arm launched with {world} ranks)"},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": s.cores, "kind": "port",
                         "sample": s.describe()},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ----------------------------------------------------------------------------- main
def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["l8_decode", "y34_decode"], default="l8_decode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the paged / shard / serving sub-benches")
    ap.add_argument("--no-prefill", action="store_true", help="skip the config-3 prefill contract object")
    ap.add_argument("--unfused", action="store_true", help="separate kv_append + decode launches per layer")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps eagerly (no CUDA graph)")
    ap.add_argument("--gather", choices=["none", "fused", "nccl"], default="none",
                    help="N>1: all-gather the output heads every layer (fused peer-memory kernel or NCCL)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup()

    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0

    res = bench_decode(args, world, rank, local)
    if rank == 0:
        cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(args.workload, world)
        line = {
            "metric": res.pop("metric"), "value": res.pop("value"), "unit": res.pop("unit"),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res.pop("ms_per_step"), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded randn K/V/Q)",
            "config": {"workload": res.pop("workload"), "parallelism": f"tp{world}-kv-heads",
                       "l2": "inputs larger than L2 (1 GiB K+V per layer)", **res.pop("geometry")},
            "roofline": res.pop("roofline"),
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": res.pop("e2e"), "clocks": res.pop("clocks"), "gpu_launches": res.pop("gpu_launches"),
            **res,
        }
        if world == 1 and not args.no_prefill:
            try:
                line["prefill"] = bench_prefill(local, cpu=not args.no_cpu_baseline)
            except Exception as e:   # must not void the headline line
                line["prefill"] = {"error": repr(e)[:300]}
        if not args.no_extras and world == 1:
            extras = {}
            for name, fn in (("decode_growth", extra_decode_growth), ("prefill_paged", extra_prefill),
                             ("long_prefill", extra_long_prefill), ("varlen_prefill", extra_varlen_prefill),
                             ("paged_vs_contiguous", extra_paged), ("long_decode", extra_long_decode),
                             ("y34_shards", extra_y34_shards), ("l8_shards", extra_l8_shards),
                             ("libraries", extra_libraries),
                             ("serving", extra_serving)):
                try:
                    extras[name] = fn(local)
                except Exception as e:   # an extra must not void the headline line
                    extras[name] = {"error": repr(e)[:300]}
            line["extras"] = extras
            # the BASELINE metric "exposed map ms/iter" in one place: steady decode (headline run),
            # decode growth across page-groups, and the config-5 serving trace
            g, sv = extras.get("decode_growth", {}), extras.get("serving", {})
            line["exposed_map_ms_per_iter_summary"] = {
                "steady_decode": line.get("exposed_map_ms_per_iter"),
                "decode_growth_sync": g.get("sync", {}).get("exposed_map_ms_per_iter"),
                "decode_growth_reference_overlap": g.get("overlapped", {}).get("exposed_map_ms_per_iter"),
                "decode_growth_prefetch_worker": g.get("overlapped_prefetch64", {}).get("exposed_map_ms_per_iter"),
                "serving_reference_overlap": sv.get("overlapped", {}).get("exposed_map_ms_per_iter"),
                "serving_sync_chunk4": sv.get("sync_chunk4", {}).get("exposed_map_ms_per_iter"),
                "serving_reference_overlap_chunk4": sv.get("overlapped_chunk4", {}).get("exposed_map_ms_per_iter"),
                "serving_staged_chunk4": sv.get("overlapped_staged_chunk4", {}).get("exposed_map_ms_per_iter"),
                "serving_staged_chunk4_p99": sv.get("overlapped_staged_chunk4", {}).get("exposed_map_ms_p99"),
                "serving_paged_layout_host": sv.get("paged_bs16", {}).get("exposed_map_ms_per_iter"),
            }
            # config-5 end to end: tokens/s of each vAttention loop over the paged-layout loop
            pg = sv.get("paged_bs16", {}).get("tokens_per_s")
            if pg:
                line["serving_tokens_per_s_vs_paged"] = {
                    k: round(v["tokens_per_s"] / pg, 3) for k, v in sv.items()
                    if isinstance(v, dict) and v.get("tokens_per_s") and k != "paged_bs16"}
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
