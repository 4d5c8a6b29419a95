"""KV append > L2 (4 requests x 16K tokens, Yi-6B KV heads, 256 MiB moved) and the 16K single
prompt: us per launch with an L2 flush before each; run under VATTN_APPEND_UNROLL / _BPS."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import kv_append
from paper_2405_04437_b200.geometry import yi_6b
MB2 = 2 << 20
dev = torch.device("cuda")
S, R = 16384, 4
g = yi_6b(max_context=S, max_batch=R)
g = g.__class__(**{**g.to_dict(), "n_layers": 1})
mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(R * 2 * 17 + 8) * MB2))
rids = [mgr.alloc_reqid() for _ in range(R)]
assert mgr.step([S] * R).ok
kn = torch.randn(R, S, 4, 128, device=dev, dtype=torch.bfloat16); vn = torch.randn_like(kn)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
idx = torch.tensor(rids, dtype=torch.int32, device=dev)
zeros = torch.zeros(R, dtype=torch.int32, device=dev)
res = {}
for name, (k, v, z, ix) in {"4x16k": (kn, vn, zeros, idx), "1x16k": (kn[:1], vn[:1], zeros[:1], idx[:1])}.items():
    times = []
    for it in range(25):
        flush.sum()                    # read-based L2 flush
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); kv_append(mgr, 0, k, v, z, ix); e1.record(); torch.cuda.synchronize()
        if it >= 5: times.append(e0.elapsed_time(e1) * 1e3)
    us = sorted(times)[len(times) // 2]
    nbytes = 2 * 2 * k.numel() * 1
    res[name] = f"{us:.1f} us {2 * k.numel() * 2 * 2 / us / 1e3:.0f} GB/s"
print(os.environ.get("VATTN_APPEND_UNROLL", "1"), os.environ.get("VATTN_APPEND_BPS", "8"), res)
mgr.close()
