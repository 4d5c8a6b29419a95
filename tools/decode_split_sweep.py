"""Decode split-K sweep on B200 (HBM GB/s by num_splits); four distinct caches are cycled so a
shape smaller than L2 is still read from HBM, as in a multi-layer step."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits
dev = torch.device("cuda")
shapes = [(64, 4, 1, 4096), (64, 8, 2, 4096), (64, 16, 4, 4096), (64, 32, 8, 4096),
          (128, 7, 1, 8192), (128, 14, 2, 8192), (16, 32, 8, 16384), (1, 32, 4, 16384)]
if len(sys.argv) > 1 and sys.argv[1] == "all":
    shapes += [(128, 56, 8, 8192), (128, 28, 4, 8192)]
for (B, hq, hkv, L) in shapes:
    kv = [(torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * hkv * 128 * 2
    res = {}
    for s in (1, 2, 3, 4, 6, 8, 12, 16):
        for i in range(4):
            decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(16):
            decode_attention_raw(q, kv[i % 4][0], kv[i % 4][1], seq, num_splits=s)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 16
        res[s] = round(byt / us / 1e3)
    best = max(res, key=res.get)
    print(f"B={B} hq={hq} hkv={hkv} L={L}: GB/s by splits {res} best={best} auto={decode_num_splits(B, hkv, L)}",
          flush=True)
    del kv
