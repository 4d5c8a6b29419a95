"""Persistent varlen prefill (VATTN_PF_PERSIST=1) vs the one-CTA-per-item kernel: bit-equal
outputs on several prompt mixes, and timings.  Each setting runs in its own process."""
import os, subprocess, sys, json

CHILD = r'''
import sys, json, torch, hashlib
sys.path.insert(0, ".")
from paper_2405_04437_b200.attention import prefill_attention_varlen_raw
dev = torch.device("cuda")
cases = {"16x512": [512] * 16, "32x256": [256] * 32, "8x2048": [2048] * 8,
         "mixed": [100, 700, 1500, 3000, 64, 2048, 1, 333], "prefix": [300, 1000, 17],
         "64x128": [128] * 64, "4x3072": [3072] * 4, "2x8192": [8192] * 2, "1x16384": [16384],
         "serve8": [2900, 180, 1210, 2400, 640, 3050, 95, 1777], "noncausal": [200, 900, 1600, 40] * 4}
res = {}
later = []
for name, lens in cases.items():
    n = len(lens)
    L = max(lens) + (512 if name == "prefix" else 0)
    g = torch.Generator(device=dev).manual_seed(n * 7 + L)
    k = torch.randn(n, L, 8, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(n, L, 8, 128, device=dev, dtype=torch.bfloat16, generator=g)
    tot = sum(lens)
    q = torch.randn(tot, 32, 128, device=dev, dtype=torch.bfloat16, generator=g)
    o = torch.empty_like(q)
    kvl = [l + (512 if name == "prefix" else 0) for l in lens]
    call = lambda: prefill_attention_varlen_raw(q, k, v, lens, list(range(n)), kv_lens=kvl, out=o,
                                                causal=(name != "noncausal"))
    for _ in range(3): call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): call()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    res[name] = {"us": us, "sha": hashlib.sha1(o.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16],
                 "finite": bool(torch.isfinite(o.float()).all())}
    if name in ("mixed", "prefix", "noncausal"):    # a few requests against the fp32 oracle, after
        offs = [0]                                  # the timings (CPU work perturbs them)
        for l in lens: offs.append(offs[-1] + l)
        later.append((name, [(q[offs[i]:offs[i + 1]].cpu(), k[i, :kvl[i]].cpu(), v[i, :kvl[i]].cpu(),
                              o[offs[i]:offs[i + 1]].cpu()) for i in (0, 1, len(lens) - 1)]))
from oracle.attention import prefill_ref, max_rel_err
for name, reqs in later:
    res[name]["oracle_err"] = max(max_rel_err(oo, prefill_ref(qq, kk, vv, causal=(name != "noncausal")))
                                  for qq, kk, vv, oo in reqs)
print("RESULT " + json.dumps(res))
'''

def run(persist, headpair=None):
    env = dict(os.environ, VATTN_PF_PERSIST=str(persist))
    if headpair is not None:
        env["VATTN_PF_HEADPAIR"] = str(headpair)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    for line in r.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    print(r.stdout[-2000:], r.stderr[-3000:])
    return None

if "--headpair" in sys.argv:
    # 2 x 2: grid / persistent x row tiles / head pairs (Params::head_pair); all bit-equal to grid+rows
    sets = {(pe, hp): run(pe, hp) for pe in (0, 1) for hp in (0, 1)}
    base = sets[(0, 0)]
    ok = all(r is not None for r in sets.values())
    print(f"{'case':10s}" + "".join(f"{'persist' if pe else 'grid'}+{'heads' if hp else 'rows':6s} us   " for pe, hp in sets))
    for k in base:
        row = f"{k:10s}"
        for key, r in sets.items():
            same = r[k]["sha"] == base[k]["sha"]
            oe = r[k].get("oracle_err")
            ok &= same and r[k]["finite"] and (oe is None or oe <= 2e-2)
            row += f"{r[k]['us']:11.1f}{'' if same else '!'}     "
        best = min(sets, key=lambda kk: sets[kk][k]["us"])
        row += f"best {best}  x{base[k]['us'] / sets[best][k]['us']:.2f} vs grid+rows"
        print(row)
    print("ALL BIT-EQUAL" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)

quick = "--quick" in sys.argv
a, b = run(0), run(1)
ok = True
for k in a:
    same = a[k]["sha"] == b[k]["sha"]
    ok &= same and b[k]["finite"]
    oe = b[k].get("oracle_err")
    if oe is not None:
        ok &= oe <= 2e-2
    print(f"{k:8s} grid {a[k]['us']:8.1f} us   persistent {b[k]['us']:8.1f} us   x{a[k]['us'] / b[k]['us']:.2f}   "
          f"bit-equal {same}" + (f"   oracle max_rel_err {oe:.2e}" if oe is not None else ""))
print("ALL BIT-EQUAL" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
