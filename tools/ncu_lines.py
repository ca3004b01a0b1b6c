"""Aggregate ncu warp-stall samples per CUDA source line:  python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
func = None
data = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not func or not re.search(kre, func):
        continue
    if len(r) < 5 or not r[0].isdigit():
        continue
    si = 4
    try:
        n = int(r[si])
    except ValueError:
        continue
    data[(func, int(r[0]))] = (n, r[1])
tot = sum(v[0] for v in data.values()) or 1
for (f, ln), (n, src) in sorted(data.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{n:7d} {100.0 * n / tot:5.1f}%  L{ln:<5d} {src.strip()[:110]}")
print("total samples", tot)
