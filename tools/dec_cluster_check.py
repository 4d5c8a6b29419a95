"""Decode split-K: the in-cluster DSMEM combine (default) vs the combine kernel
(VATTN_DEC_CLUSTER=0).  Prints one line per case with a checksum of the bf16 output bits and the
max-normalised error against the fp32 oracle; run once per mode and compare the checksums."""
import os, sys
sys.path.insert(0, ".")
import torch
from oracle.attention import decode_ref, max_rel_err
from paper_2405_04437_b200.attention import decode_attention_raw, decode_attention_append_raw

dev = torch.device("cuda")
for B, hq, hkv, D, L, S in ((3, 32, 8, 128, 1000, 2), (2, 8, 2, 64, 3000, 3), (4, 32, 8, 128, 5000, 5), (1, 32, 8, 128, 32768, 16), (2, 32, 8, 128, 20000, 12),
                            (1, 32, 8, 128, 32768, 8), (64, 4, 1, 128, 4097, 2), (2, 56, 8, 128, 700, 8)):
    g = torch.Generator(device=dev).manual_seed(B * 1000 + S)
    kc = torch.randn(B, L + 8, hkv, D, device=dev, dtype=torch.bfloat16, generator=g)
    vc = torch.randn(B, L + 8, hkv, D, device=dev, dtype=torch.bfloat16, generator=g)
    q = torch.randn(B, hq, D, device=dev, dtype=torch.bfloat16, generator=g)
    seq = torch.randint(L // 2, L + 1, (B,), device=dev, generator=g, dtype=torch.int32)
    seq[0] = 0 if B > 2 else seq[0]           # an empty row: every split empty
    out = decode_attention_raw(q, kc, vc, seq, num_splits=S)
    kn = torch.randn(B, hkv, D, device=dev, dtype=torch.bfloat16, generator=g)
    out2 = decode_attention_append_raw(q, kc, vc, kn, kn, seq, num_splits=S)
    torch.cuda.synchronize()
    ref = decode_ref(q.cpu(), kc.cpu(), vc.cpu(), seq.cpu())
    h = (out.view(torch.int16).to(torch.int64) * torch.arange(out.numel(), device=dev).view_as(out).remainder(7919)).sum().item()
    h2 = (out2.view(torch.int16).to(torch.int64) * torch.arange(out2.numel(), device=dev).view_as(out2).remainder(7919)).sum().item()
    print(f"case B{B} hq{hq} hkv{hkv} D{D} L{L} S{S}: sig {h} {h2} err {max_rel_err(out.cpu(), ref):.2e}", flush=True)
