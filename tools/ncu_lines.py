"""Per CUDA source line of an ncu report: warp-stall samples, warp instructions executed, shared-memory
wavefronts (and ideal), average active threads.

    python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top] [sort: samples|inst|smem]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = sys.argv[4] if len(sys.argv) > 4 else "samples"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
func, hdr, data = None, None, {}


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not func or not re.search(kre, func):
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    data[(func, int(r[0]))] = (num(r[4]), num(d.get("Instructions Executed")), num(d.get("L1 Wavefronts Shared")),
                               num(d.get("L1 Wavefronts Shared Ideal")), num(d.get("Avg. Threads Executed")), r[1])
idx = {"samples": 0, "inst": 1, "smem": 2}[key]
tot = [sum(v[i] for v in data.values()) or 1 for i in range(3)]
print(f"{'samples':>8} {'%':>5} {'warp-inst':>10} {'%':>5} {'smem-wf':>9} {'ideal':>9} {'thr':>5}  line")
for (f, ln), v in sorted(data.items(), key=lambda kv: -kv[1][idx])[:top]:
    print(f"{v[0]:8.0f} {100 * v[0] / tot[0]:5.1f} {v[1]:10.0f} {100 * v[1] / tot[1]:5.1f} {v[2]:9.0f} {v[3]:9.0f} "
          f"{v[4]:5.1f}  L{ln:<5d} {v[5].strip()[:90]}")
print("totals: samples %.0f  warp-inst %.0f  smem wavefronts %.0f" % tuple(tot))
