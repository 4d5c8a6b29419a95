"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, both at once on two
streams (the prefill e2e pipeline's bound)."""
import torch
dev = torch.device("cuda")
n = 160 << 20
hi = torch.empty(n, dtype=torch.uint8).pin_memory()
ho = torch.empty(128 << 20, dtype=torch.uint8).pin_memory()
di = torch.empty(n, dtype=torch.uint8, device=dev)
do = torch.empty(128 << 20, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
def h2d():
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
a, b, c = timed(h2d), timed(d2h), timed(both)
print(f"H2D 160 MiB {a:.2f} ms = {n / a / 1e6:.1f} GB/s; D2H 128 MiB {b:.2f} ms = {(128 << 20) / b / 1e6:.1f} GB/s; "
      f"both concurrently {c:.2f} ms (sum {a + b:.2f}, max {max(a, b):.2f})")
