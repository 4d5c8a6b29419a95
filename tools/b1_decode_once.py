"""B 1 x 32K decode (Llama-3-8B heads) for ncu launch lists: 6 calls at the automatic split."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw
dev = torch.device("cuda")
B, L = 1, 32768
kv = [(torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16),
       torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16)) for _ in range(2)]
q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
seq = torch.full((B,), L, dtype=torch.int32, device=dev)
for i in range(6):
    decode_attention_raw(q, kv[i % 2][0], kv[i % 2][1], seq)
torch.cuda.synchronize()
