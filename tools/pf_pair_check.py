"""Correctness + speed of the CTA-pair prefill kernel (VATTN_PF_PAIR=1) against torch SDPA (fp32
math on the GPU) and the single-CTA kernel; run each mode in its own process:
    VATTN_PF_PAIR=1 python tools/pf_pair_check.py"""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_raw

dev = torch.device("cuda")
mode = "pair" if os.environ.get("VATTN_PF_PAIR", "0") == "1" else "single"
for S, hq, hkv, kv in ((256, 32, 4, 256), (512, 8, 2, 600), (1000, 32, 8, 1000), (3000, 32, 4, 3100), (4096, 32, 8, 4096)):
    g = torch.Generator(device=dev).manual_seed(S)
    k = torch.randn(1, kv, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(1, kv, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16, generator=g)
    out = prefill_attention_raw(q, k, v, 0, kv)
    torch.cuda.synchronize()
    # reference: fp32, causal aligned bottom-right (query i sees keys <= i + kv - S)
    qf = q.float().permute(1, 0, 2)
    kf = k[0].float().permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
    vf = v[0].float().permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
    s = torch.matmul(qf, kf.transpose(1, 2)) / 128 ** 0.5
    mask = torch.arange(kv, device=dev).view(1, -1) > (torch.arange(S, device=dev).view(-1, 1) + kv - S)
    s.masked_fill_(mask, float("-inf"))
    ref = torch.matmul(torch.softmax(s, -1), vf).permute(1, 0, 2)
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"{mode} S={S} hq={hq} hkv={hkv} kv={kv}: max-normalised err {err:.2e} {'OK' if err <= 2e-2 else 'FAIL'}", flush=True)
for S, hq, hkv in (() if "--parity-only" in sys.argv else ((16384, 32, 4), (4096, 32, 8), (65536, 32, 4))):
    k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
    q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    n = 3 if S > 20000 else 10
    for _ in range(3): prefill_attention_raw(q, k, v, 0, S, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): prefill_attention_raw(q, k, v, 0, S, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{mode} S={S}: {ms:.3f} ms {2.0 * S * S * 128 * hq / ms / 1e9:.0f} TFLOP/s", flush=True)
