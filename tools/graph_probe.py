"""Host launch overhead vs GPU time of the decode step at the per-GPU shard shapes of a
KV-head-sharded job (G = 1, 2, 4, 8 on one GPU): eager per-layer launches vs one CUDA-graph
replay of the 32-layer fused append+decode."""
import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append
from paper_2405_04437_b200.geometry import llama3_8b

MB2 = 2 << 20
dev = torch.device("cuda")
res = {}
for G in (1, 2, 4, 8):
    g = llama3_8b(max_context=8192, max_batch=64).with_tp(G)
    B, N, hq, hkv, d = g.max_batch, g.n_layers, g.q_heads_per_worker, g.kv_heads_per_worker, g.head_dim
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=6 * 2 * N * B * MB2, eager_groups=0,
                                          reclaim_threshold=0.0), backend="cuda", device=0)
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([4200] * B).ok
    q = torch.randn(N, B, hq, d, device=dev, dtype=torch.bfloat16)
    kn = torch.randn(N, B, hkv, d, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    pos = torch.full((B,), 4096, dtype=torch.int32, device=dev)

    def layers():
        for layer in range(N):
            decode_attention_append(mgr, layer, q[layer], kn[layer], kn[layer], pos, idx, out=out[layer])

    for _ in range(3):
        layers()
    torch.cuda.synchronize()
    # eager: host wall per step and device time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        layers()
    e1.record()
    host_eager = (time.perf_counter() - t0) / 20 * 1e3
    torch.cuda.synchronize()
    dev_eager = e0.elapsed_time(e1) / 20
    # graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
        layers()
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        graph.replay()
    e1.record()
    host_graph = (time.perf_counter() - t0) / 20 * 1e3
    torch.cuda.synchronize()
    dev_graph = e0.elapsed_time(e1) / 20
    ref = out.clone()
    layers()
    torch.cuda.synchronize()
    res[f"G{G}"] = {"host_ms_per_step_eager": round(host_eager, 3), "device_ms_per_step_eager": round(dev_eager, 3),
                    "host_ms_per_step_graph": round(host_graph, 3), "device_ms_per_step_graph": round(dev_graph, 3),
                    "graph_equals_eager": bool(torch.equal(ref, out))}
    print(G, res[f"G{G}"], flush=True)
    del graph
    mgr.close()
json.dump(res, open("gpurun_out/graph_probe.json", "w"), indent=1)
