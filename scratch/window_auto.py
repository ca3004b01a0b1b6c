"""auto window width per config: chosen w, error vs an accurate NFFT (w=8, os=8), time"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
from paper_2401_08260_b200 import inputs as I
dev = torch.device("cuda", 0)
for name, Nsc in [("cfg1", None), ("cfg3", None), ("cfg4", None), ("cfg5", 2_000_000), ("paper_gauss", None),
                  ("paper_matern", None), ("paper_laplace", None)]:
    cfg = I.CONFIGS[name]
    if Nsc: cfg = I.scaled(cfg, N=Nsc, M=Nsc)
    x, y, w = (torch.from_numpy(a).to(dev) for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    par = I.kernel_param(cfg)
    sw = float(w.abs().sum())
    ref = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, window_w=8, oversample=8, engine="nfft").double()
    s = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p).double()
    pl = S.sks_last_plan()
    s6 = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, window_w=6).double()
    print(json.dumps({"cfg": name, "w_auto": pl["window_w"], "err_auto": float((s - ref).abs().max()) / sw,
                      "err_w6": float((s6 - ref).abs().max()) / sw}), flush=True)
