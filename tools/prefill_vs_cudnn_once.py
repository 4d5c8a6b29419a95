"""One launch each of our prefill and cuDNN SDPA on the Y6 16K shape (for ncu comparison)."""
import sys
sys.path.insert(0, ".")
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel
from paper_2405_04437_b200.attention import prefill_attention_raw
dev = torch.device("cuda")
S, hq, hkv, d = 16384, 32, 4, 128
kc = torch.randn(1, S, hkv, d, device=dev, dtype=torch.bfloat16); vc = torch.randn_like(kc)
qp = torch.randn(S, hq, d, device=dev, dtype=torch.bfloat16)
qh = qp.transpose(0, 1).unsqueeze(0)
kh = kc[0].repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0)
vh = vc[0].repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0)
for _ in range(2):
    prefill_attention_raw(qp, kc, vc, 0, S)
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True)
torch.cuda.synchronize()
