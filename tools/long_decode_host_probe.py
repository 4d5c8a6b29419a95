"""Is few-row long-context decode host-bound?  B 1 x L, Llama-3-8B heads: eager event timing
vs host enqueue time per call vs the same calls replayed from a CUDA graph."""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits

dev = torch.device("cuda")
for B, L in ((1, 32768), (1, 131072), (8, 32768)):
    kv = [(torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    outs = [torch.empty(B, 32, 128, device=dev, dtype=torch.bfloat16) for _ in range(4)]
    byt = 2 * B * L * 8 * 128 * 2

    def run8():
        for i in range(8):
            decode_attention_raw(q, kv[i % 4][0], kv[i % 4][1], seq, out=outs[i % 4])

    for _ in range(3):
        run8()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    run8()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) * 1e3 / 8
    host = (t1 - t0) * 1e6 / 8
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run8()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run8()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) * 1e3 / 32
    print(f"B{B} L{L} splits {decode_num_splits(B, 8, L)}: eager {eager:.1f} us ({byt / eager / 1e3:.0f} GB/s), "
          f"host enqueue {host:.1f} us/call, graph {graph:.1f} us ({byt / graph / 1e3:.0f} GB/s)", flush=True)
    del kv
    torch.cuda.empty_cache()
