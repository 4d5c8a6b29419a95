"""Per-CTA timeline of a short-prompt varlen prefill launch (trace build, -DVATTN_PF_TRACE):
16 x 512 and 8 x 2048 Llama-3-8B-head prompts.  Fixed per-CTA cost vs per-KV-tile cost, gaps
between consecutive CTAs on an SM, and the tail."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2405_04437_b200._abi import LIB_PATH
from paper_2405_04437_b200.attention import prefill_attention_varlen_raw
raw = C.CDLL(str(LIB_PATH))
dev = torch.device("cuda")
for n_req, S in ((16, 512), (8, 2048)):
    k = torch.randn(n_req, S, 8, 128, device=dev, dtype=torch.bfloat16); v = torch.randn_like(k)
    q = torch.randn(n_req * S, 32, 128, device=dev, dtype=torch.bfloat16)
    o = torch.empty_like(q)
    call = lambda: prefill_attention_varlen_raw(q, k, v, [S] * n_req, list(range(n_req)), out=o)
    for _ in range(3): call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); call(); e1.record(); torch.cuda.synchronize()
    buf = np.zeros((8192, 12), dtype=np.uint64)
    raw.vattn_debug_prefill_cta(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    n = 32 * n_req * ((S + 255) // 256)
    b = buf[:n].astype(np.int64)
    t0 = b[:, 0].min(); st, en, sm, kv = b[:, 0] - t0, b[:, 1] - t0, b[:, 2], b[:, 3]
    dur = en - st
    span = en.max()
    A = np.vstack([np.ones(n), kv]).T
    (a, c), *_ = np.linalg.lstsq(A, dur, rcond=None)
    gaps = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        o_ = np.argsort(st[idx])
        ss, ee = st[idx][o_], en[idx][o_]
        gaps += list(ss[1:] - ee[:-1])
    gaps = np.array(gaps)
    print(f"{n_req}x{S}: event {e0.elapsed_time(e1)*1e3:.1f} us, CTA span {span/1e3:.1f} us, {n} CTAs on {len(np.unique(sm))} SMs")
    print(f"  CTA duration: mean {dur.mean()/1e3:.2f} us, kv tiles mean {kv.mean():.1f}; fit fixed {a/1e3:.2f} us + {c:.0f} ns per KV tile")
    print(f"  gap between CTAs on an SM: mean {gaps.mean()/1e3:.2f} us, p50 {np.median(gaps)/1e3:.2f}, p90 {np.percentile(gaps, 90)/1e3:.2f}")
    ent, pro, ext, pre = b[:, 4] - t0, b[:, 5] - t0, b[:, 6] - t0, b[:, 7] - t0
    print(f"  t0: end->after fence {np.mean(b[:, 8] - t0 - en)/1e3:.2f}, end->after barrier {np.mean(b[:, 9] - t0 - en)/1e3:.2f};"
          f" warp9: end->at fence {np.mean(b[:, 10] - t0 - en)/1e3:.2f} us")
    print(f"  end of work -> before dealloc {np.mean(pre - en)/1e3:.2f} us; dealloc {np.mean(ext - pre)/1e3:.2f} us")
    print(f"  entry -> work item known {np.mean(st - ent)/1e3:.2f} us; entry -> prologue done {np.mean(pro - ent)/1e3:.2f} us;"
          f" end of work -> TMEM released {np.mean(ext - en)/1e3:.2f} us")
    lg = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        o_ = np.argsort(ent[idx])
        lg += list(ent[idx][o_][1:] - ext[idx][o_][:-1])
    lg = np.array(lg)
    print(f"  TMEM released -> next CTA's first instruction on the SM: mean {lg.mean()/1e3:.2f} us, p50 {np.median(lg)/1e3:.2f}")
    print(f"  first CTA start to last start {st.max()/1e3:.1f} us; tail after last start {(span - st.max())/1e3:.1f} us")
