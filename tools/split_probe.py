"""Fixed vs per-token cost of the decode kernel at the L8/G8 shard shape (64 rows x 1 KV head):
run under ncu --metrics gpu__time_duration.sum; seqlen 64..4096, 1 split."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw
dev = torch.device("cuda")
B, hq, hkv = 64, 4, 1
for L in (64, 256, 1024, 2048, 4096):
    kv = [(torch.randn(B, max(L, 64), hkv, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, max(L, 64), hkv, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    for i in range(4):
        decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=1)
    torch.cuda.synchronize()
    del kv
