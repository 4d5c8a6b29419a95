"""Timeline of one heavy prefill CTA (build with VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE): softmax busy /
wait per tile and the MMA issuer's own durations (P wait, PV issue, S issue).  Y6 16K causal.
Run the variant under test with VATTN_PF_VAR."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2405_04437_b200._abi import LIB_PATH
from paper_2405_04437_b200.attention import prefill_attention_raw
raw = C.CDLL(str(LIB_PATH))
dev = torch.device("cuda")
S, hq, hkv = 16384, 32, 4
k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
for _ in range(3): prefill_attention_raw(q, k, v, 0, S)
torch.cuda.synchronize()
buf = np.zeros((4, 160, 8), dtype=np.uint64)
raw.vattn_debug_prefill_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
b = buf.astype(np.int64)
J = range(10, 120)
sm_busy = [b[0, j, 2] - b[0, j, 1] for j in J]
sm_wait = [b[0, j + 1, 1] - b[0, j, 2] for j in J]
period = [b[0, j + 1, 1] - b[0, j, 1] for j in J]
p_lat = [b[2, j, 1] - b[0, j, 2] for j in J]              # softmax P arrive -> issuer sees P
pv_iss = [b[2, j, 2] - b[2, j, 1] for j in J]              # 8 PV MMAs issued
s_iss = [b[2, j, 3] - b[2, j, 2] for j in J]               # K wait + 8 S MMAs issued + commit
s_lat = [b[0, j + 1, 1] - b[2, j, 3] for j in J]           # S issued -> softmax sees S(j+1)
fine = {}
for (ea, eb, name) in ((1, 3, "S got -> first half computed"), (3, 4, "vote + first P stored (issued)"),
                     (4, 5, "second half computed"), (5, 6, "vote + second P stored (issued)"),
                     (6, 7, "tcgen05.wait::st"), (7, 2, "fence + arrive")):
    v_ = [d_ for d_ in (int(b[0, j, eb]) - int(b[0, j, ea]) for j in J) if 0 < d_ < 100000]
    if v_:
        print(f"  {name:36s} mean {np.mean(v_):7.0f}")
for name, v_ in (("softmax A busy", sm_busy), ("softmax A wait for next S", sm_wait), ("period", period),
                 ("P arrive -> issuer wakes", p_lat), ("PV issue (8 MMA)", pv_iss), ("S issue (8 MMA + commit)", s_iss),
                 ("S issue done -> softmax got S", s_lat)):
    print(f"{name:32s} mean {np.mean(v_):7.0f}  p10 {np.percentile(v_, 10):7.0f}  p90 {np.percentile(v_, 90):7.0f}")
