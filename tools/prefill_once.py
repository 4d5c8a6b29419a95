import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_raw
dev = torch.device("cuda")
import os
S, hq, hkv = int(os.environ.get("PF_S", 16384)), 32, 4
k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16); out = torch.empty_like(q)
for _ in range(4):
    prefill_attention_raw(q, k, v, 0, S, out=out)
torch.cuda.synchronize()
