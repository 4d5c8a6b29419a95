"""Why is cuMemSetAccess slower inside the decode-growth loop (bench extra decode_growth) than in
isolation (vmm_load_probe)?  Sync-mode growth loop variants; per-call driver costs of the maps
issued by step() during the loop."""
import json, math, statistics, sys, time
sys.path.insert(0, ".")
import ctypes as C
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append
from paper_2405_04437_b200.geometry import llama3_8b

MB2 = 2 << 20
dev = torch.device("cuda")
g = llama3_8b(max_context=8192, max_batch=64)
B, N = g.max_batch, g.n_layers
tok = g.per_token_layer_bytes
gen = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(N, B, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
kn = torch.randn(N, B, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
out = torch.empty_like(q)


def run(name, kernels=True, layers=N, sync_each=True, sleep_ms=0.0, steps=64, stagger=16, pre_create=1.0,
        bg=False, wait="sync", prefetch=0):
    ctx0 = [3584 + stagger * b for b in range(B)]
    groups = max(math.ceil((c + steps + 4) * tok / MB2) for c in ctx0)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(groups + 1) * 2 * N * B * MB2,
                                          eager_groups=0, reclaim_threshold=0.0, pre_create_fraction=pre_create),
                         backend="cuda", device=0, prefetch_tokens=prefetch)
    rids = [mgr.alloc_reqid() for _ in range(B)]
    seq = [0] * B
    for r, c in zip(rids, ctx0):
        seq[r] = c
    assert mgr.step(seq).ok
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    pos = torch.tensor([seq[r] for r in rids], dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    st0 = mgr.driver_stats()
    per, ex = [], []
    for it in range(steps):
        nxt = [s + 1 for s in seq]
        s0 = mgr.driver_stats(peek=True)
        t0 = time.perf_counter()
        assert mgr.step(nxt).ok
        dt = time.perf_counter() - t0
        ex.append(dt * 1e3)
        s1 = mgr.driver_stats(peek=True)
        n = s1["real_set_access_calls"] - s0["real_set_access_calls"]
        if n:
            per.append(((s1["real_set_access_wall_us"] - s0["real_set_access_wall_us"]) / n, n, dt * 1e3))
        if kernels:
            for layer in range(layers):
                decode_attention_append(mgr, layer, q[layer], kn[layer], kn[layer], pos, idx, out=out[layer])
        pos.add_(1)
        seq = nxt
        if bg:
            mgr.bg_submit(mgr.plan_overlap([x + 1 for x in seq]), prefetch=prefetch > 0)
        if sync_each:
            if wait == "sync":
                torch.cuda.synchronize()
            else:                      # poll an event without blocking inside the driver
                ev = torch.cuda.Event()
                ev.record()
                while not ev.query():
                    time.sleep(50e-6)
        if sleep_ms:
            time.sleep(sleep_ms / 1e3)
    torch.cuda.synchronize()
    if bg:
        mgr.bg_wait()
    st = mgr.driver_stats()
    mgr.close()
    n = st["real_set_access_calls"] - st0["real_set_access_calls"]
    r = {"exposed_ms_mean": round(statistics.mean(ex), 3), "exposed_ms_max": round(max(ex), 2),
         "set_access_us_per_call": round((st["real_set_access_wall_us"] - st0["real_set_access_wall_us"]) / max(1, n), 1),
         "calls": n, "bursts_us_per_call": [round(p[0]) for p in per], "burst_step_ms": [round(p[2], 1) for p in per]}
    print(name, r, flush=True)
    return r


res = {}
for rep in range(2):
    res[f"C_kernels_sync_{rep}"] = run(f"C_kernels_sync_{rep}")
    res[f"O1_bg_sync_{rep}"] = run(f"O1_bg_sync_{rep}", bg=True)
    res[f"O4_bg_prefetch64_sync_{rep}"] = run(f"O4_bg_prefetch64_sync_{rep}", bg=True, prefetch=64)
    res[f"O6_bg_prefetch128_sync_{rep}"] = run(f"O6_bg_prefetch128_sync_{rep}", bg=True, prefetch=128)
json.dump(res, open("gpurun_out/growth_probe3.json", "w"), indent=1)
