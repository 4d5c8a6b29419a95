"""Does background cuMemMap/cuMemSetAccess serialize with GPU work / host CUDA calls on B200?"""
import json, sys, time, threading
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry

MB2 = 2 * 1024 * 1024
dev = torch.device("cuda")
g = ModelGeometry(32, 8, 128, 2, max_context=4096, max_batch=8, n_q_heads_total=32)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
res = {}

def fresh():
    m = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=8 * 4 * 64 * MB2))
    for _ in range(8):
        m.alloc_reqid()
    return m

def plan_for(m, groups):
    nxt = [groups * 1024] * 8
    return m.plan_overlap(nxt)

def run(mode, groups=1):
    m = fresh()
    m.step([1] * 8)              # 1 group mapped per slot (sync)
    plan = plan_for(m, 1 + groups)
    n_pages = len(plan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m.bg_submit(plan)
    if mode == "idle":
        time.sleep(0.05)
    elif mode == "gemm_sync":           # long GPU work, host blocked in synchronize
        for _ in range(40):
            a @ a
        torch.cuda.synchronize()
    elif mode == "small_kernels":       # many short launches + syncs (decode-like)
        x = torch.randn(1024, device=dev)
        for i in range(2000):
            x.mul_(1.0001)
            if i % 50 == 0:
                torch.cuda.synchronize()
    elif mode == "gemm_nosync":         # GPU busy, host not calling CUDA
        for _ in range(40):
            a @ a
        time.sleep(0.3)
    main_s = time.perf_counter() - t0
    r = m.bg_wait()
    torch.cuda.synchronize()
    st = m.driver_stats()
    m.close()
    return {"pages": n_pages, "bg_wall_ms": round(r.bg_wall_us / 1e3, 2), "main_ms": round(main_s * 1e3, 1),
            "us_per_page": round(r.bg_wall_us / max(1, n_pages), 1),
            "map_us_per_page": round(st["real_map_wall_us"] / max(1, st["real_maps"]), 2),
            "setaccess_us_per_call": round(st["real_set_access_wall_us"] / max(1, st["real_set_access_calls"]), 1)}

# warm
torch.cuda.synchronize(); (a @ a); torch.cuda.synchronize()
for mode in ["idle", "gemm_sync", "gemm_nosync", "small_kernels", "idle"]:
    res[mode] = run(mode)
    print(mode, res[mode], flush=True)
