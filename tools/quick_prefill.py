import sys, time
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_raw
dev = torch.device("cuda")
for S, hq, hkv in ((16384, 32, 4), (8192, 32, 8), (4096, 32, 8)):
    k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
    q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    for _ in range(3): prefill_attention_raw(q, k, v, 0, S, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): prefill_attention_raw(q, k, v, 0, S, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = 2.0 * S * S * 128 * hq
    print(f"prefill S={S} hq={hq} hkv={hkv}: {ms:.3f} ms  {fl/ms/1e9:.0f} TFLOP/s (causal 2*S^2*D*H)")
