import os, subprocess, sys
res = {}
for rep in range(2):
    for pp in ("0", "1"):
        r = subprocess.run([sys.executable, "tools/quick_prefill.py"], env=dict(os.environ, VATTN_PF_POLY=pp),
                           capture_output=True, text=True)
        lines = r.stdout.splitlines()
        res.setdefault(pp, []).append([l.split()[-4] for l in lines] if lines else r.stderr[-200:])
for k, v in res.items():
    print("poly", k, "TFLOP/s at 16K/8K/4K:", v)
