"""Host enqueue cost of one decode call, split into the Python wrapper and the C ABI call
(B 1 x 32K, Llama-3-8B heads; no synchronisation inside the timed loops)."""
import ctypes as C
import math
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2405_04437_b200.attention import _workspace, cache_desc, decode_attention_raw
from paper_2405_04437_b200._abi import lib

dev = torch.device("cuda")
B, L = 1, 32768
k = torch.randn(B, L, 8, 128, device=dev, dtype=torch.bfloat16)
v = torch.randn_like(k)
q = torch.randn(B, 32, 128, device=dev, dtype=torch.bfloat16)
seq = torch.full((B,), L, dtype=torch.int32, device=dev)
out = torch.empty_like(q)
for _ in range(5):
    decode_attention_raw(q, k, v, seq, out=out)
torch.cuda.synchronize()


def host_us(fn, n=200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


desc = cache_desc(k, v)
ws = _workspace(dev, lib().vattn_decode_workspace_bytes(B, 32, 128, 0))
args = (C.byref(desc), C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()), B, 32, C.c_void_p(seq.data_ptr()), None,
        1.0 / math.sqrt(128), 0, C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream))
print(f"python wrapper + C ABI: {host_us(lambda: decode_attention_raw(q, k, v, seq, out=out)):.1f} us/call")
print(f"C ABI call only:        {host_us(lambda: lib().vattn_decode_raw(*args)):.1f} us/call")
print(f"cache_desc only:        {host_us(lambda: cache_desc(k, v)):.1f} us/call")
