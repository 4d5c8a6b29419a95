"""Host cost of one cuTensorMapEncodeTiled (the varlen prefill encodes two per request per call)."""
import ctypes as C
import time

import torch

torch.cuda.init()
cu = C.CDLL("libcuda.so.1")
buf = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
m = (C.c_uint8 * 128)()
dims = (C.c_uint64 * 3)(128, 8, 4096)
strides = (C.c_uint64 * 2)(256, 2048)
box = (C.c_uint32 * 3)(64, 1, 128)
es = (C.c_uint32 * 3)(1, 1, 1)
f = cu.cuTensorMapEncodeTiled
f.restype = C.c_int
args = lambda: (C.byref(m), 10, 3, C.c_void_p(buf.data_ptr()), dims, strides, box, es, 0, 3, 2, 0)
assert f(*args()) == 0, f(*args())
n = 20000
t0 = time.perf_counter()
for _ in range(n):
    f(*args())
t1 = time.perf_counter()
print(f"cuTensorMapEncodeTiled via ctypes: {(t1 - t0) / n * 1e6:.2f} us per call (includes ~0.5-1 us ctypes overhead)")
