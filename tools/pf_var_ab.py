"""A/B of prefill kernel variants (VATTN_PF_VAR bits, pf::VAR_* in csrc/prefill.cu) on one GPU.

    python tools/pf_var_ab.py [vars...]        (default 0 1 3 4 5 7), two interleaved rounds

Each variant runs in its own process (the variant is read once per process); outputs are
compared bit for bit against variant 0 on the same seeded inputs."""
import os, subprocess, sys, json

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2405_04437_b200.attention import prefill_attention_raw
dev = torch.device("cuda")
res = {}
for S, hq, hkv in ((16384, 32, 4), (4096, 32, 8), (65536, 32, 4)):
    g = torch.Generator(device=dev).manual_seed(S)
    k = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(1, S, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    q = torch.randn(S, hq, 128, device=dev, dtype=torch.bfloat16, generator=g)
    out = torch.empty_like(q)
    n = 3 if S > 20000 else 10
    for _ in range(3): prefill_attention_raw(q, k, v, 0, S, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): prefill_attention_raw(q, k, v, 0, S, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 2.0 * S * S * 128 * hq
    h = out.view(torch.int16).to(torch.int64)
    res[f"S{S}"] = {"ms": ms, "tflops": fl / ms / 1e9, "sig": int((h * torch.arange(h.numel(), device=dev).view_as(h).remainder(9973)).sum().item())}
print("RESULT " + json.dumps(res))
'''

def run(var):
    env = dict(os.environ, VATTN_PF_VAR=str(var))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    for line in r.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    return {"error": (r.stderr or r.stdout)[-800:]}

vars_ = [int(x) for x in sys.argv[1:]] or [0, 1, 3, 4, 5, 7]
allres = {}
for rnd in range(2):
    for v in vars_:
        res = run(v)
        allres.setdefault(v, []).append(res)
        print(f"round {rnd} var {v}: " + json.dumps({k: (round(x['tflops'], 1) if 'tflops' in x else x) for k, x in res.items()} if "error" not in res else res), flush=True)
base = allres.get(vars_[0], [{}])[0]
for v, rs in allres.items():
    same = all(rs[0].get(k, {}).get("sig") == base.get(k, {}).get("sig") for k in base if "sig" in base[k])
    print(f"var {v}: bit-equal to var {vars_[0]}: {same}")
