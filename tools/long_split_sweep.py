"""Split-K sweep for few-row long-context decode (B 1-4, Llama-3-8B heads): GB/s by num_splits."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits
dev = torch.device("cuda")
for (B, L) in ((1, 32768), (1, 131072), (2, 65536), (4, 32768), (8, 32768)):
    kv = [(torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * 8 * 128 * 2
    res = {}
    for s in (2, 4, 8, 16, 19, 24, 32, 37, 48, 64):
        for i in range(4):
            decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(16):
            decode_attention_raw(q, kv[i % 4][0], kv[i % 4][1], seq, num_splits=s)
        e1.record(); torch.cuda.synchronize()
        res[s] = round(byt / (e0.elapsed_time(e1) * 1e3 / 16) / 1e3)
    print(f"B={B} L={L}: GB/s by splits {res} auto={decode_num_splits(B, 8, L)}", flush=True)
    del kv
