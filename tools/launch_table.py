"""Per-kernel table from an ncu --csv launch list:  python tools/launch_table.py launches.csv [first_id]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = (int(d["ID"]), d["Kernel Name"].split("(")[0][-40:], d["Grid Size"])
    data.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, nm, g), m in sorted(data.items()):
    if i < first:
        continue
    print(f"{i:>4} {nm:40s} {g:>16s} {m.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us"
          + (f"  dram r {m['dram__bytes_read.sum'] / 1e6:8.1f} MB w {m['dram__bytes_write.sum'] / 1e6:8.1f} MB"
             if "dram__bytes_read.sum" in m else ""))
