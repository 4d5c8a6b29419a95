"""Few-row long-context decode: does filling all 148 SMs (splits = floor(148 / units)) beat the
128-CTA target of auto_splits?  Graph-replayed (no host enqueue), four cache copies cycled so
every call reads HBM; Llama-3-8B heads (32 Q / 8 KV, D 128).  Prints GB/s per split count."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits

dev = torch.device("cuda")
out = {}
for B, L, splits in ((1, 32768, (16,)), (2, 65536, (0, 8, 9)), (3, 32768, (0, 5, 6)), (4, 32768, (0, 3, 4)), (2, 32768, (0, 8, 9)), (6, 16384, (0, 3, 4)),
                     (5, 32768, (0, 3, 4)), (7, 16384, (0, 2, 3))):
    ncopy = 4
    kv = [(torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16)) for _ in range(ncopy)]
    q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    byt = 2 * B * L * 8 * 128 * 2
    row = {"auto": decode_num_splits(B, 8, L)}
    ref = None
    for s in splits:
        for i in range(ncopy):
            decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=s)
        torch.cuda.synchronize()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st, capture_error_mode="thread_local"):
            for i in range(ncopy):
                o = decode_attention_raw(q, kv[i][0], kv[i][1], seq, num_splits=s)
        gr.replay()
        torch.cuda.synchronize()
        if ref is None:
            ref = o.float().clone()
        err = (o.float() - ref).abs().max().item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            for _ in range(4):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / (4 * ncopy))
        row[s] = {"us": round(best, 2), "gbs": round(byt / (best * 1e-6) / 1e9), "maxdiff_vs_first": err}
        del gr
    out[f"B{B}_L{L}"] = row
    print(f"B={B} L={L}: " + json.dumps(row), flush=True)
    del kv
