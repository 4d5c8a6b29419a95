"""The headline step's shape (Llama-3-8B, B 64, ctx 4096 + 1 appended, 32 layers) replayed from one
CUDA graph: VMM cache with 2 MiB handles vs 8 MiB chunks vs 32 plain cudaMalloc layers; ms per
step and per layer, no L2 flush (32 GiB of K/V streams past L2 anyway)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append, decode_attention_append_raw
from paper_2405_04437_b200.geometry import llama3_8b

dev = torch.device("cuda")
MB2 = 2 << 20
B, N, hq, hkv, d = 64, 32, 32, 8, 128
q = torch.randn(N, B, hq, d, device=dev, dtype=torch.bfloat16)
kn = torch.randn(N, B, hkv, d, device=dev, dtype=torch.bfloat16)
o = torch.empty_like(q)
pos = torch.full((B,), 4096, dtype=torch.int32, device=dev)


def run(body, label):
    body()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cap, capture_error_mode="thread_local"):
        body()
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): gr.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{label}: {ms:.3f} ms/step {ms / N * 1e3:.1f} us/layer {N * 2 * B * 4097 * hkv * d * 2 / ms / 1e9:.0f} GB/s", flush=True)


for chunk in [int(x) for x in (sys.argv[1:] or ["1", "4"])]:
    g = llama3_8b(max_context=4160, max_batch=B)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * N * B * 5 + 8) * MB2), phys_chunk_groups=chunk)
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([4100] * B).ok
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    run(lambda: ([decode_attention_append(mgr, l, q[l], kn[l], kn[l], pos, idx, out=o[l]) for l in range(N)], mgr.mark_use()),
        f"VMM cache, phys_chunk_groups={chunk}")
    mgr.close()
    torch.cuda.empty_cache()
ks = [torch.zeros(B, 4160, hkv, d, device=dev, dtype=torch.bfloat16) for _ in range(N)]
vs = [torch.zeros(B, 4160, hkv, d, device=dev, dtype=torch.bfloat16) for _ in range(N)]
run(lambda: [decode_attention_append_raw(q[l], ks[l], vs[l], kn[l], kn[l], pos, out=o[l]) for l in range(N)],
    "plain cudaMalloc layers (raw API)")
