import os, subprocess, sys
code = r'''
import sys; sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw
dev = torch.device("cuda")
for (B, hq, hkv, L) in ((64, 32, 8, 4096), (128, 56, 8, 8192), (128, 7, 1, 8192), (16, 32, 8, 16384)):
    k = torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
    q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * hkv * 128 * 2
    best = 0
    for s in (1, 2):
        for _ in range(3): decode_attention_raw(q, k, v, seq, num_splits=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): decode_attention_raw(q, k, v, seq, num_splits=s)
        e1.record(); torch.cuda.synchronize()
        gbs = byt / (e0.elapsed_time(e1) * 50) / 1e3
        print(f"  B={B} hq={hq} hkv={hkv} L={L} splits={s}: {gbs:.0f} GB/s", flush=True)
    del k, v
'''
for st in ("4", "3", "2"):
    print("stages", st, flush=True)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, VATTN_DEC_STAGES=st), capture_output=True, text=True)
    print(r.stdout or r.stderr[-400:], flush=True)
