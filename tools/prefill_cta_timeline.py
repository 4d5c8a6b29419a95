"""Per-CTA timeline of one Y6 16K (and 4K) causal prefill launch (trace build): how much of the
kernel's SM-time is CTA work proportional to its KV tiles, fixed per-CTA cost, gaps between CTAs
on an SM, and the tail."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2405_04437_b200._abi import LIB_PATH
from paper_2405_04437_b200.attention import prefill_attention_raw
raw = C.CDLL(str(LIB_PATH))
dev = torch.device("cuda")
for S, hq, hkv in ((16384, 32, 4), (4096, 32, 8)):
    k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
    q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
    for _ in range(3): prefill_attention_raw(q, k, v, 0, S)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); prefill_attention_raw(q, k, v, 0, S); e1.record(); torch.cuda.synchronize()
    buf = np.zeros((8192, 12), dtype=np.uint64)
    raw.vattn_debug_prefill_cta(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    n = hq * ((S + 255) // 256)
    b = buf[:n].astype(np.int64)
    t0 = b[:, 0].min(); st, en, sm, kv = b[:, 0] - t0, b[:, 1] - t0, b[:, 2], b[:, 3]
    dur = en - st
    span = en.max()
    # per-tile cost from a least-squares fit dur = a + c * kv
    A = np.vstack([np.ones(n), kv]).T
    (a, c), *_ = np.linalg.lstsq(A, dur, rcond=None)
    busy = np.zeros(sm.max() + 1)
    for i in range(n): busy[sm[i]] += dur[i]
    used = busy[busy > 0]
    print(f"S={S}: event {e0.elapsed_time(e1)*1e3:.1f} us, CTA span {span/1e3:.1f} us, {n} CTAs on {len(used)} SMs")
    print(f"  fit: per-CTA fixed {a/1e3:.2f} us + {c:.0f} ns per KV tile (ideal tile at period 3160 cyc / 1.965 GHz = {3160/1.965:.0f} ns)")
    print(f"  SM busy: mean {used.mean()/1e3:.1f} us, min {used.min()/1e3:.1f}, max {used.max()/1e3:.1f} (of span {span/1e3:.1f})")
    print(f"  fixed share of SM-time: {n*a/used.sum():.3f}; idle share (span*SMs - busy): {1 - used.sum()/(span*len(used)):.3f}")
    first_end = np.sort(en)[:148].max()
    print(f"  last CTA starts at {st.max()/1e3:.1f} us; tail after the last start: {(span - st.max())/1e3:.1f} us")
