"""Window width / oversampling sweep: error vs an accurate NFFT (w=8, os=8, eps=1e-10) and time, per config."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S  # noqa: E402
from paper_2401_08260_b200 import inputs as I  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dev = torch.device("cuda", 0)
for name, Nsc in [("cfg4", None), ("cfg5", 2_000_000), ("paper_gauss", None),
                  ("paper_matern", None)]:
    cfg = I.CONFIGS[name]
    if Nsc:
        cfg = I.scaled(cfg, N=Nsc, M=Nsc)
    x, y, w = (torch.from_numpy(a).to(dev) for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    par = I.kernel_param(cfg)
    sw = float(w.abs().sum())
    ref = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, window_w=8,
                    oversample=8, engine="nfft").double()
    for ww in (4, 6, 8):
        for os_ in (2, 4, 8):
            kw = dict(window_w=ww, oversample=os_, engine="nfft")
            s = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, **kw).double()
            err = float((s - ref).abs().max()) / sw
            ms = timed(lambda: S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, **kw))
            pl = S.sks_last_plan()
            print(json.dumps({"cfg": name, "N": cfg.N, "w": ww, "os": os_, "n": pl.get("n"), "err": err, "ms": ms}),
                  flush=True)
