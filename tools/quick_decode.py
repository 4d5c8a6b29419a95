"""Quick decode/append timing on the L8 shape (development aid, not the bench)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_attention_paged, kv_append_raw, decode_num_splits

dev = torch.device("cuda")
B, hq, hkv, d, L = 64, 32, 8, 128, 4096
k = torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)
v = torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)
q = torch.randn(B, hq, d, device=dev, dtype=torch.bfloat16)
seq = torch.full((B,), L, dtype=torch.int32, device=dev)
byt = 2 * B * L * hkv * d * 2 + 2 * B * hq * d * 2
for splits in [0, 1, 2, 3, 4, 6, 8]:
    for _ in range(3):
        decode_attention_raw(q, k, v, seq, num_splits=splits)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        decode_attention_raw(q, k, v, seq, num_splits=splits)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / n
    print(f"decode splits={splits} (auto={decode_num_splits(B, hkv, L)}): {us:.1f} us  {byt/us/1e3:.0f} GB/s")
# paged
for bs in (16, 256):
    maxb = L // bs
    kp = k.view(B * maxb, bs, hkv, d); vp = v.view(B * maxb, bs, hkv, d)
    bt = torch.randperm(B * maxb, device=dev).view(B, maxb).to(torch.int32)
    for _ in range(3):
        decode_attention_paged(q, kp, vp, bt, seq)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        decode_attention_paged(q, kp, vp, bt, seq)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20
    print(f"paged bs={bs}: {us:.1f} us {byt/us/1e3:.0f} GB/s")
# append prefill-size
S = 16384
kc = torch.empty(1, S, 4, d, device=dev, dtype=torch.bfloat16); vc = torch.empty_like(kc)
kn = torch.randn(1, S, 4, d, device=dev, dtype=torch.bfloat16); vn = torch.randn_like(kn)
z = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(3): kv_append_raw(kc, vc, kn, vn, z)
torch.cuda.synchronize()
e0.record()
for _ in range(20): kv_append_raw(kc, vc, kn, vn, z)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1000 / 20
print(f"append 16K x 4 x 128: {us:.1f} us {4*S*4*d*2/us/1e3:.0f} GB/s")
