"""B 1 x 32K / 128K decode (8 KV heads, 16 splits), graph-replayed, under the current env
(VATTN_DEC_CLUSTER16, VATTN_DEC_CW, VATTN_DEC_STAGES, VATTN_DEC_SPLITS)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import decode_attention_raw
dev = torch.device("cuda")
res = {}
for L in (32768, 131072):
    kv = [(torch.randn(1, L, 8, 128, device=dev, dtype=torch.bfloat16), torch.randn(1, L, 8, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(1, 32, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((1,), L, dtype=torch.int32, device=dev)
    ref = decode_attention_raw(q, kv[0][0], kv[0][1], seq, num_splits=1)
    for i in range(4): decode_attention_raw(q, kv[i][0], kv[i][1], seq)
    torch.cuda.synchronize()
    chk = decode_attention_raw(q, kv[0][0], kv[0][1], seq)
    err = ((chk.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
    cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
        for i in range(4): decode_attention_raw(q, kv[i][0], kv[i][1], seq)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 40
    res[L] = f"{us:.1f} us {2 * L * 8 * 128 * 2 / us / 1e3:.0f} GB/s err-vs-unsplit {err:.1e}"
print({k: os.environ.get(k, "-") for k in ("VATTN_DEC_CLUSTER16", "VATTN_DEC_CW", "VATTN_DEC_STAGES", "VATTN_DEC_SPLITS")}, res)
