import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw
dev = torch.device("cuda")
for (B, hq, hkv, L, s) in ((64, 4, 1, 4096, 2), (64, 4, 1, 2048, 1), (64, 4, 1, 4096, 1), (128, 4, 1, 2048, 1)):
    kv = [(torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16), torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    for i in range(8):
        decode_attention_raw(q, kv[i % 4][0], kv[i % 4][1], seq, num_splits=s)
    torch.cuda.synchronize()
    del kv
