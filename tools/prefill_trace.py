import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2405_04437_b200._abi import lib, LIB_PATH
from paper_2405_04437_b200.attention import prefill_attention_raw
raw = C.CDLL(str(LIB_PATH))
dev = torch.device("cuda")
S, hq, hkv = 16384, 32, 4
k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
for _ in range(3): prefill_attention_raw(q, k, v, 0, S)
torch.cuda.synchronize()
buf = np.zeros((4, 160, 4), dtype=np.uint64)
raw.vattn_debug_prefill_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
t0 = int(buf[0, 0, 0])
for j in list(range(0, 8)) + list(range(60, 66)) + list(range(124, 128)):
    a = [int(x) - t0 if x else -1 for x in buf[0, j, :3]]
    b = [int(x) - t0 if x else -1 for x in buf[1, j, :3]]
    ma = [int(x) - t0 if x else -1 for x in buf[2, j, :2]]
    mb = [int(x) - t0 if x else -1 for x in buf[3, j, :2]]
    print(f"j={j:3d} smA wait>{a[0]:8d} got {a[1]:8d} P {a[2]:8d} (T_s={a[2]-a[1]:5d}) | smB got {b[1]:8d} P {b[2]:8d} (T_s={b[2]-b[1]:5d}) | mmaA waitP {ma[0]:8d}->{ma[1]:8d} | mmaB waitP {mb[0]:8d}->{mb[1]:8d}")
# averages over the middle
ts_a = [int(buf[0, j, 2]) - int(buf[0, j, 1]) for j in range(10, 120)]
idle_a = [int(buf[0, j + 1, 1]) - int(buf[0, j, 2]) for j in range(10, 120)]
per = [(int(buf[0, j + 1, 1]) - int(buf[0, j, 1])) for j in range(10, 120)]
print("mean softmax A busy", np.mean(ts_a), "mean A wait for next S", np.mean(idle_a), "period", np.mean(per))
