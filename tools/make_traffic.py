"""profiles/traffic_<cfg>.json from an ncu --csv launch list with dram__bytes_read.sum / dram__bytes_write.sum:
per kernel slot of bench.py, the DRAM bytes (read + write) of all the slot's kernel launches in one call (calls =
k_finalize launches); bench.py divides by the slot's timed scopes per call.

    python tools/make_traffic.py launches.csv cfg2 > profiles/traffic_cfg2.json
"""
import csv
import json
import sys

SLOTS = [("k_split3", "split3"), ("k_proj_tc", "project"), ("k_proj_pair", "project"), ("k_minmax", "minmax"), ("k_prep_f16", "minmax"),
         ("k_sample_mean", "minmax"), ("k_bound_ranges", "minmax"),
         ("k_sp_hist", "sp_hist"), ("k_sp_part", "sp_part"), ("k_sp_owner", "sp_owner"), ("k_sp_gather", "sp_gather"),
         ("k_plan", "plan"), ("k_proj_spread", "spread"), ("k_spread", "spread"), ("k_fft_filter", "fft_filter"),
         ("k_proj_eval", "eval"), ("k_eval", "eval")]
rows = list(csv.reader(open(sys.argv[1])))
hdr, per = None, {}
# complete calls only: launches up to the last k_finalize (a launch list cut by ncu -c may end inside a call)
fin = [int(r[0]) for r in rows if len(r) > 4 and r[0].isdigit() and "k_finalize" in r[4]]
last = max(fin) if fin else 1 << 60
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) or not r[0].isdigit() or int(r[0]) > last:
        continue
    d = dict(zip(hdr, r))
    slot = next((s for k, s in SLOTS if k in d["Kernel Name"]), None)
    if slot is None or d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    per.setdefault(slot, {}).setdefault(d["ID"], 0.0)
    per[slot][d["ID"]] += float(d["Metric Value"].replace(",", ""))
calls = len({r[0] for r in rows if len(r) > 4 and "k_finalize" in r[4]}) or 1
out = {s: sum(v.values()) / calls for s, v in per.items()}
# the sort stage (bench.py slot "sortsum"): all its kernel launches of one call
if "sp_hist" in per:
    out["sortsum"] = sum(sum(per[k].values()) for k in ("sp_hist", "sp_part", "sp_owner", "sp_gather") if k in per) / calls
out["_source"] = f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({sys.argv[2]}); bytes per call, cold L2"
print(json.dumps(out, indent=1))
