"""Summarise an ncu SASS source-page CSV: per-opcode totals and hottest instructions.

    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv; python tools/sass_hot.py x.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
col = {n: i for i, n in enumerate(hdr)}
data = rows[2:]


def f(r, name):
    try:
        return float(r[col[name]] or 0)
    except (KeyError, ValueError):
        return 0.0


tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
by_op = defaultdict(lambda: [0.0, 0.0])
for r in data:
    op = r[col["Source"]].split()[0] if r[col["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += f(r, "Instructions Executed")
    by_op[op][1] += f(r, "Warp Stall Sampling (All Samples)")
print(f"total instr {tot_i:.3e}  samples {tot_s:.0f}")
for op, (i, s) in sorted(by_op.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{op:12s} instr {i / tot_i * 100:6.2f}%  stalls {s / tot_s * 100:6.2f}%")
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(f(r, c) for r in data) for c in stall_cols}
print("stall reasons:", ", ".join(f"{c[6:]} {v / tot_s * 100:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
print("hottest instructions:")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = max(stall_cols, key=lambda c: f(r, c))
    print(f"  {r[col['Address']]:>6s} {f(r, 'Warp Stall Sampling (All Samples)') / tot_s * 100:5.2f}% {top[6:]:14s} {r[col['Source']][:90]}")
