"""Short-prompt varlen prefill (Llama-3-8B heads): event-timed call vs the kernel alone.
Run under ncu for the kernel's own duration; without ncu it prints the event-timed figure."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2405_04437_b200.attention import prefill_attention_varlen_raw
dev = torch.device("cuda")
for n_req, S in ((16, 512), (32, 256), (8, 2048)):
    k = torch.randn(n_req, S, 8, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    q = torch.randn(n_req * S, 32, 128, device=dev, dtype=torch.bfloat16)
    o = torch.empty_like(q)
    call = lambda: prefill_attention_varlen_raw(q, k, v, [S] * n_req, list(range(n_req)), out=o)
    for _ in range(3): call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): call()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    # host cost of one call with the GPU idle
    import time
    t = time.perf_counter()
    for _ in range(20): call()
    host = (time.perf_counter() - t) / 20 * 1e3
    torch.cuda.synchronize()
    fl = n_req * 2.0 * S * S * 128 * 32
    print(f"{n_req}x{S}: event {ms*1e3:.1f} us/call ({fl/ms/1e9:.0f} TF), host enqueue {host*1e3:.1f} us/call")

# host cost of one call with an idle GPU (synchronize between calls)
import time
for n_req, S in ((16, 512), (32, 256), (8, 2048), (1, 512)):
    k = torch.randn(n_req, S, 8, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    q = torch.randn(n_req * S, 32, 128, device=dev, dtype=torch.bfloat16)
    o = torch.empty_like(q)
    call = lambda: prefill_attention_varlen_raw(q, k, v, [S] * n_req, list(range(n_req)), out=o)
    for _ in range(3): call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t = time.perf_counter(); call(); ts.append(time.perf_counter() - t); torch.cuda.synchronize()
    ts.sort()
    print(f"{n_req}x{S}: host per call (GPU idle) p50 {ts[10]*1e6:.1f} us")
