"""L8 layer (B 64, 8 KV heads, D 128): plain decode over 4096 / 4097 rows vs fused append+decode
(appends row 4096, attends over 4097), raw API, back-to-back launches (1 GiB per layer > L2)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_attention_append_raw

dev = torch.device("cuda")
B, hq, hkv, d, L = 64, 32, 8, 128, 4160
k = torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)
v = torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)
q = torch.randn(B, hq, d, device=dev, dtype=torch.bfloat16)
kn = torch.randn(B, hkv, d, device=dev, dtype=torch.bfloat16)


def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


for n_rows in (4096, 4097, 4160):
    seq = torch.full((B,), n_rows, dtype=torch.int32, device=dev)
    us = timeit(lambda: decode_attention_raw(q, k, v, seq))
    print(f"plain decode over {n_rows} rows: {us:.1f} us {2 * B * n_rows * hkv * d * 2 / us / 1e3:.0f} GB/s")
seq = torch.full((B,), 4096, dtype=torch.int32, device=dev)
us = timeit(lambda: decode_attention_append_raw(q, k, v, kn, kn, seq))
print(f"fused append+decode (row 4096, over 4097): {us:.1f} us {2 * B * 4097 * hkv * d * 2 / us / 1e3:.0f} GB/s")

# the same layer on the VMM-backed cache (2 MiB page-groups), manager API and raw views
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append
from paper_2405_04437_b200.geometry import llama3_8b
MB2 = 2 << 20
for chunk in (1, 4):
    g = llama3_8b(max_context=4160, max_batch=B)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * B * 5 + 8) * MB2), phys_chunk_groups=chunk)
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([4100] * B).ok
    kc, vc = mgr.k_cache(0), mgr.v_cache(0)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    for r in range(B):
        kc[rids[r], :4096].copy_(k[r, :4096]); vc[rids[r], :4096].copy_(v[r, :4096])
    torch.cuda.synchronize()
    us = timeit(lambda: decode_attention_append(mgr, 0, q, kn, kn, seq, idx))
    print(f"chunk{chunk} manager fused append+decode: {us:.1f} us {2 * B * 4097 * hkv * d * 2 / us / 1e3:.0f} GB/s")
    us = timeit(lambda: decode_attention_append_raw(q, kc, vc, kn, kn, seq, idx))
    print(f"chunk{chunk} raw fused on the VMM views: {us:.1f} us {2 * B * 4097 * hkv * d * 2 / us / 1e3:.0f} GB/s")
    mgr.close()
