"""Is a slow box slow at reading?  HBM copy (read+write) vs read-only streaming (torch max /
sum reductions over 4 GiB) vs the L8 decode kernel (4 cache copies cycled), on the same box."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw

dev = torch.device("cuda")


def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev).normal_()
b = torch.empty_like(a)
print("copy  GB/s", round(2 * a.numel() * 2 / t(lambda: b.copy_(a)) / 1e6))
big = torch.empty(1 << 31, dtype=torch.bfloat16, device=dev).normal_()
print("amax  GB/s", round(big.numel() * 2 / t(lambda: big.amax()) / 1e6))
print("sum   GB/s", round(big.numel() * 2 / t(lambda: big.sum()) / 1e6))
del a, b, big
B, hq, hkv, d, L = 64, 32, 8, 128, 4096
kv = [(torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16), torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
q = torch.randn(B, hq, d, device=dev, dtype=torch.bfloat16)
seq = torch.full((B,), L, dtype=torch.int32, device=dev)
byt = 2 * B * L * hkv * d * 2
i = [0]


def dec():
    k, v = kv[i[0] % 4]; i[0] += 1
    decode_attention_raw(q, k, v, seq)


print("decode GB/s", round(byt / t(dec, 20) / 1e6))
