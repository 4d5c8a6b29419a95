import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_raw
dev = torch.device("cuda")
S = int(sys.argv[1]); L = int(sys.argv[2]); slots = int(sys.argv[3]); slot = int(sys.argv[4])
k = torch.randn(slots, L, 4, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
q = torch.randn(S, 32, 128, device=dev, dtype=torch.bfloat16)
out = prefill_attention_raw(q, k, v, slot, S)
torch.cuda.synchronize(); print("raw ok", S, L, slots, slot, flush=True)
