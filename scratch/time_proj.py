"""time sks_project on a (scaled) config's points (x and y stacked)"""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
from paper_2401_08260_b200 import inputs as I
name, _, n = sys.argv[1].partition(":")
cfg = I.CONFIGS[name]
if n: cfg = I.scaled(cfg, N=int(n), M=int(n))
dev = torch.device("cuda", 0)
pts = torch.cat([torch.from_numpy(I.points(cfg, "x")), torch.from_numpy(I.points(cfg, "y"))]).to(dev)
for _ in range(2): z = S.sks_project(pts, cfg.P, cfg.dir_seed)
torch.cuda.synchronize()
del z
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); z = S.sks_project(pts, cfg.P, cfg.dir_seed); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b)); del z
print(json.dumps({"cfg": sys.argv[1], "emode": os.environ.get("SKS_PROJ_EMODE", "0"), "ms": sorted(ts)}))
