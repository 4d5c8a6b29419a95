import sys, os
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
from paper_2405_04437_b200.attention import kv_append, prefill_attention
dev = torch.device("cuda")
g = ModelGeometry(2, 4, 128, 2, max_context=4096, max_batch=2, n_q_heads_total=32)
mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 * 1024 * 1024, pool_bytes=64 * 2 * 1024 * 1024))
r0, r1 = mgr.alloc_reqid(), mgr.alloc_reqid()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
lens = [0, 0]; lens[r1] = S
print("step", mgr.step(lens), mgr.slots, flush=True)
print("bases", [hex(b.device_ptr) for b in mgr.buffers], mgr.slot_stride, flush=True)
kn = torch.randn(1, S, 4, 128, device=dev).to(torch.bfloat16); vn = torch.randn_like(kn)
q = torch.randn(S, 32, 128, device=dev).to(torch.bfloat16)
kv_append(mgr, 1, kn, vn, torch.zeros(1, dtype=torch.int32, device=dev), torch.tensor([r1], dtype=torch.int32, device=dev))
torch.cuda.synchronize(); print("append ok", flush=True)
kc = mgr.k_cache(1); print("view", kc.shape, kc.stride(), float(kc[r1, :S].float().sub(kn[0].float()).abs().max()), flush=True)
out = prefill_attention(mgr, 1, q, r1)
torch.cuda.synchronize(); print("prefill ok", flush=True)
