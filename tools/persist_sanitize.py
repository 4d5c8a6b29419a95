"""Small persistent-varlen prefill launch for compute-sanitizer (memcheck / synccheck)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_varlen_raw
dev = torch.device("cuda")
lens = [256, 100, 384, 1, 300, 256, 129, 512] * 4
n = len(lens)
k = torch.randn(n, 512, 8, 128, device=dev, dtype=torch.bfloat16)
v = torch.randn_like(k)
q = torch.randn(sum(lens), 32, 128, device=dev, dtype=torch.bfloat16)
o = prefill_attention_varlen_raw(q, k, v, lens, list(range(n)))
torch.cuda.synchronize()
print("finite", bool(torch.isfinite(o.float()).all()))
