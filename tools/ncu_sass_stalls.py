"""Summarise an ncu `--page source --csv --print-source sass` export: stall samples by reason,
by opcode, and the hottest instructions.  python tools/ncu_sass_stalls.py file.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
def num(x):
    try: return float(x)
    except ValueError: return 0.0
tot = collections.Counter(); by_op = collections.Counter(); ex_op = collections.Counter()
for r in data:
    op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
    if op.startswith("@"): op = r[col["Source"]].split()[1]
    op = op.split(".")[0]
    s = num(r[col["Warp Stall Sampling (All Samples)"]])
    by_op[op] += s
    ex_op[op] += num(r[col["Instructions Executed"]])
    for h in stall_cols: tot[h] += num(r[col[h]])
T = sum(tot.values())
print(f"total samples {T:.0f}")
for h, v in tot.most_common(12): print(f"  {h:28s} {v/T*100:5.1f}%")
print("samples by opcode (top 20) / warp-instructions executed")
for op, v in by_op.most_common(20): print(f"  {op:12s} {v/T*100:5.1f}%   exec {ex_op[op]:.3e}")
print("total warp instructions executed", sum(ex_op.values()))
print(f"hottest {top} instructions")
hot = sorted(data, key=lambda r: -num(r[col["Warp Stall Sampling (All Samples)"]]))[:top]
for r in hot:
    s = num(r[col["Warp Stall Sampling (All Samples)"]])
    reasons = sorted(((num(r[col[h]]), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"  {r[0][-5:]} {s/T*100:5.2f}% {r[col['Source']].strip()[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in reasons if v))
