"""Split count vs bandwidth for grids that leave SMs idle (units = batch x KV heads < 148), timed
from CUDA-graph replays (no host pacing).  VATTN_DEC_STAGES may force the TMA ring depth."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2405_04437_b200.attention import decode_attention_raw, decode_num_splits

dev = torch.device("cuda")
cases = ((64, 4, 1, 4096), (4, 32, 8, 32768), (1, 32, 8, 32768), (16, 32, 8, 8192))
for B, hq, hkv, L in cases:
    kv = [(torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16),
           torch.randn(B, L, hkv, 128, device=dev, dtype=torch.bfloat16)) for _ in range(4)]
    q = torch.randn(B, hq, 128, device=dev, dtype=torch.bfloat16)
    seq = torch.full((B,), L, dtype=torch.int32, device=dev)
    outs = [torch.empty(B, hq, 128, device=dev, dtype=torch.bfloat16) for _ in range(4)]
    byt = 2 * B * L * hkv * 128 * 2
    units = B * hkv
    res = {}
    for s in sorted({1, 2, 3, 4, 5, 6, 8, 9, 12, 16, 18, 24, 32, 37}):
        if s * units > 4 * 148 or (s > 1 and L // s < 256):
            continue

        def run8():
            for i in range(8):
                decode_attention_raw(q, kv[i % 4][0], kv[i % 4][1], seq, out=outs[i % 4], num_splits=s)

        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            run8()
        torch.cuda.current_stream().wait_stream(st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run8()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 32
        res[s] = (round(us, 1), round(byt / us / 1e3))
        del g
    print(f"B{B} hq{hq} hkv{hkv} L{L} (units {units}, auto {decode_num_splits(B, hkv, L)}): "
          + ", ".join(f"s{s}: {u} us {gb} GB/s" for s, (u, gb) in res.items()), flush=True)
    del kv
    torch.cuda.empty_cache()
