"""Map ncu SASS-page hot addresses to source lines using the cubin's line info.

    python tools/sass_lines.py <lib.so> <kernel-substring> <ncu-sass.csv> [top]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

lib, kname, csvf = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
funcs = {}
cur = None
line = None
for ln in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = {}
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        funcs[cur][int(m.group(1), 16)] = line
cands = [f for f in funcs if kname in f]
fn = sorted(cands, key=len)[0]
amap = funcs[fn]
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
col = {n: i for i, n in enumerate(hdr)}
data = rows[2:]
base = int(data[0][col["Address"]], 16)
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[col[S]] or 0) for r in data)
byline = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
for r in data:
    off = int(r[col["Address"]], 16) - base
    ln = amap.get(off, "?")
    byline[ln][0] += float(r[col[S]] or 0)
    byline[ln][1] += float(r[col["Instructions Executed"]] or 0)
    for c in stall_cols:
        byline[ln][2][c] += float(r[col[c]] or 0)
ti = sum(v[1] for v in byline.values())
print(f"function {fn}; samples {tot:.0f}")
for ln, (s, i, st) in sorted(byline.items(), key=lambda x: -x[1][0])[:top]:
    reason = max(st, key=st.get)[6:] if st else ""
    print(f"{ln:32s} stall {s / tot * 100:5.1f}%  instr {i / ti * 100:5.1f}%  top:{reason}")
