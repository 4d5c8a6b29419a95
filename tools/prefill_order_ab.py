"""A/B of the prefill grid order (VATTN_PF_HEAD_FAST=0 per-head heaviest-first, 1 global
heaviest-first with heads fastest).  `python tools/prefill_order_ab.py` runs both, interleaved."""
import os
import subprocess
import sys

sys.path.insert(0, ".")


def inner():
    import torch
    from paper_2405_04437_b200.attention import prefill_attention_raw, prefill_attention_varlen_raw

    dev = torch.device("cuda")

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for S, hq, hkv in ((4096, 32, 4), (16384, 32, 4), (65536, 32, 4)):
        k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
        v = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16)
        q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16)
        out = torch.empty_like(q)
        ms = timeit(lambda: prefill_attention_raw(q, k, v, 0, S, out=out), 3 if S > 20000 else 10)
        print(f"S{S} {2.0 * S * S * 128 * hq / ms / 1e9:.0f}")
    for n, L in ((16, 512), (8, 2048), (4, 3072)):
        k = torch.randn(n, L, 4, 128, device=dev, dtype=torch.bfloat16)
        v = torch.randn(n, L, 4, 128, device=dev, dtype=torch.bfloat16)
        q = torch.randn(n * L, 32, 128, device=dev, dtype=torch.bfloat16)
        out = torch.empty_like(q)
        ql = [L] * n
        sl = list(range(n))
        ms = timeit(lambda: prefill_attention_varlen_raw(q, k, v, ql, sl, out=out))
        print(f"V{n}x{L} {2.0 * n * L * L * 128 * 32 / ms / 1e9:.0f}")
        import time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            prefill_attention_varlen_raw(q, k, v, ql, sl, out=out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"H{n}x{L} {(t1 - t0) / 10 * 1e6:.0f}")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        inner()
        sys.exit(0)
    res = {}
    for rep in range(3):
        for hf in ("0", "1"):
            r = subprocess.run([sys.executable, __file__, "inner"], env=dict(os.environ, VATTN_PF_HEAD_FAST=hf),
                               capture_output=True, text=True)
            for line in r.stdout.splitlines():
                k, v = line.split()
                res.setdefault(k, {}).setdefault(hf, []).append(float(v))
            if r.returncode:
                print(r.stderr[-500:])
    for k, d in res.items():
        print(k, "TFLOP/s  per-head order:", d.get("0"), " heads-fast order:", d.get("1"))
