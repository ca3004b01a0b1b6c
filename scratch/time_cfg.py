"""time sks_sum on (scaled) configs: python scratch/time_cfg.py cfg5:2000000 cfg3 ..."""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
from paper_2401_08260_b200 import inputs as I
dev = torch.device("cuda", 0)
for arg in sys.argv[1:]:
    name, _, n = arg.partition(":")
    cfg = I.CONFIGS[name]
    if n: cfg = I.scaled(cfg, N=int(n), M=int(n))
    x, y, w = (torch.from_numpy(a).to(dev) for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    par = I.kernel_param(cfg)
    ws = torch.empty(S.sks_workspace_size(cfg.N, cfg.M, cfg.d, cfg.kind, par, cfg.P, 0, cfg.P, cfg.matern_p), dtype=torch.uint8, device=dev)
    f = lambda: S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, workspace=ws)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    S.sks_profile_enable(True)
    S.sks_profile_read()
    for _ in range(5): f()
    torch.cuda.synchronize()
    prof = {k: round(v[0] / 5, 4) for k, v in S.sks_profile_read().items() if v[1]}
    S.sks_profile_enable(False)
    print(json.dumps({"cfg": arg, "ms": ms, "prof": prof}), flush=True)
