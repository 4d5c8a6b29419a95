import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_attention_append_raw, kv_append_raw
dev = torch.device("cuda")
B, hq, hkv, L = 64, 32, 8, 4096
k = torch.randn(B, L + 64, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
kn = torch.randn(B, hkv, 128, device=dev, dtype=torch.bfloat16); vn = torch.randn_like(kn)
pos = torch.full((B,), L, dtype=torch.int32, device=dev); after = pos + 1
def t(fn, n=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n
for rep in range(3):
    a = t(lambda: (kv_append_raw(k, v, kn, vn, pos), decode_attention_raw(q, k, v, after)))
    b = t(lambda: decode_attention_append_raw(q, k, v, kn, vn, pos))
    c = t(lambda: decode_attention_raw(q, k, v, after))
    print(f"unfused append+decode {a:.1f} us | fused {b:.1f} us | decode only {c:.1f} us")
