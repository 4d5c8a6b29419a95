import os, subprocess, sys
res = {}
for rep in range(3):
    for pp in (0, 1, 2, 3):
        out = subprocess.run([sys.executable, "tools/quick_prefill.py"], env=dict(os.environ, VATTN_PF_POLY=str(pp)),
                             capture_output=True, text=True).stdout.splitlines()[0]
        res.setdefault(pp, []).append(float(out.split()[-4]))
for pp, v in res.items():
    print("poly", pp, "TFLOP/s at 16K:", v, "best", max(v))
