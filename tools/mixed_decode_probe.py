"""Decode over a batch of MIXED context lengths (serving-like): HBM GB/s with the auto split
count vs forced splits, against uniform lengths with the same total bytes."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits

dev = torch.device("cuda")
B, hq, hkv, d, L = 64, 32, 8, 128, 8192
gen = torch.Generator().manual_seed(0)
mixed = torch.randint(128, L + 1, (B,), generator=gen, dtype=torch.int32)
uniform = torch.full((B,), int(mixed.float().mean()), dtype=torch.int32)
kv = [(torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16), torch.randn(B, L, hkv, d, device=dev, dtype=torch.bfloat16)) for _ in range(2)]
q = torch.randn(B, hq, d, device=dev, dtype=torch.bfloat16)
for name, lens in (("uniform", uniform), ("mixed", mixed), ("mixed_sorted_desc", mixed.sort(descending=True).values)):
    seq = lens.to(dev)
    byt = 2 * int(lens.sum()) * hkv * d * 2
    res = {}
    for s in (0, 1, 2, 4, 8):
        for i in range(2):
            decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            decode_attention_raw(q, kv[i % 2][0], kv[i % 2][1], seq, num_splits=s)
        e1.record(); torch.cuda.synchronize()
        res[s] = round(byt / (e0.elapsed_time(e1) * 1e3 / 10) / 1e3)
    print(name, "GB/s by splits (0 = auto)", res, "auto =", decode_num_splits(B, hkv, L), flush=True)
