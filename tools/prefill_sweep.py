import os, subprocess, sys
res = {}
cfgs = [("1", "0"), ("1", "1"), ("2", "0"), ("2", "1"), ("2", "2")]
for rep in range(2):
    for ver, pp in cfgs:
        r = subprocess.run([sys.executable, "tools/quick_prefill.py"],
                           env=dict(os.environ, VATTN_PF_POLY=pp, VATTN_PF_VERSION=ver), capture_output=True, text=True)
        line = (r.stdout.splitlines() or [r.stderr[-200:]])[0]
        res.setdefault((ver, pp), []).append(line.split()[-4] if r.stdout else line)
for k, v in res.items():
    print("version", k[0], "poly", k[1], "TFLOP/s at 16K:", v)
