"""How does the B200 driver's cuMemSetAccess cost depend on what the GPU is doing?

One manager (Llama-3-8B shape, 64 buffers); every trial maps one page-group for 4 fresh slots
(4 x 64 = 256 maps, from pre-created handles) through execute_plan on the calling thread while
the GPU is (a) idle, (b) running a sleep kernel (busy SMs, no memory traffic), (c) streaming HBM
(large device copies), (d) running the decode kernel, and (e) idle with calls spaced 1 ms apart.
Reports µs per cuMemSetAccess / cuMemMap from the driver counters."""
import json, sys, time
sys.path.insert(0, ".")
import ctypes as C
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200._abi import lib, check
from paper_2405_04437_b200.attention import decode_attention
from paper_2405_04437_b200.geometry import llama3_8b

MB2 = 2 << 20
dev = torch.device("cuda")
g = llama3_8b(max_context=8192, max_batch=64)
B = g.max_batch
mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=6 * 64 * B * MB2, eager_groups=0,
                                      reclaim_threshold=0.0), backend="cuda", device=0)
rids = [mgr.alloc_reqid() for _ in range(B)]
seq = [1024] * B                     # one group per slot, mapped now
assert mgr.step(seq).ok
a = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
b = torch.empty_like(a)
q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
sl = torch.full((B,), 1024, dtype=torch.int32, device=dev)
idx = torch.tensor(rids, dtype=torch.int32, device=dev)
out = torch.empty_like(q)
stream = torch.cuda.current_stream()
cur = {"grp": 1}


def load(kind):
    if kind == "sleep":
        check(lib().vattn_compute_proxy(int(400e6), C.c_void_p(stream.cuda_stream)))
    elif kind == "hbm":
        for _ in range(120):          # ~0.4 s of 4 GiB/iter copies
            b.copy_(a)
    elif kind == "decode":
        for _ in range(2000):
            decode_attention(mgr, 0, q, sl, idx, out=out)


def trial(kind, slots, spaced=False):
    g0 = cur["grp"]
    nxt = list(seq)
    for r in slots:
        nxt[r] = (g0 + 1) * 1024
    plan = mgr.plan_overlap(nxt)
    torch.cuda.synchronize()
    load(kind)
    time.sleep(0.01)
    s0 = mgr.driver_stats(peek=True)
    t0 = time.perf_counter()
    if spaced:
        for e in plan:
            mgr.execute_plan([e])
            time.sleep(0.001)
    else:
        mgr.execute_plan(plan)
    wall = time.perf_counter() - t0
    s1 = mgr.driver_stats(peek=True)
    torch.cuda.synchronize()
    n = s1["real_set_access_calls"] - s0["real_set_access_calls"]
    return {"maps": s1["real_maps"] - s0["real_maps"], "set_access_calls": n,
            "set_access_us_per_call": round((s1["real_set_access_wall_us"] - s0["real_set_access_wall_us"]) / max(1, n), 1),
            "map_us_per_call": round((s1["real_map_wall_us"] - s0["real_map_wall_us"]) / max(1, s1["real_maps"] - s0["real_maps"]), 2),
            "wall_ms": round(wall * 1e3, 1)}


res = {}
order = [("idle", False), ("sleep", False), ("hbm", False), ("decode", False), ("idle", True), ("idle", False),
         ("hbm", False), ("sleep", False)]
for i, (kind, spaced) in enumerate(order):
    slots = rids[4 * i: 4 * i + 4]
    r = trial(kind, slots, spaced)
    key = f"{i}_{kind}{'_spaced' if spaced else ''}"
    res[key] = r
    print(key, r, flush=True)
mgr.close()
json.dump(res, open("gpurun_out/vmm_load_probe.json", "w"), indent=1)
