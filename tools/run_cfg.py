"""Run one configuration (optionally scaled) a few times through sks_sum and print per-kernel device times
(sks_profile_*): a small driver for ncu captures and quick A/B timings.
    python tools/run_cfg.py cfg5 [N] [M] [P] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_08260_b200 as S  # noqa: E402
from paper_2401_08260_b200 import build, inputs as I  # noqa: E402


def main():
    build.build()
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    a = [int(v) for v in sys.argv[2:]]
    cfg = I.CONFIGS[name]
    kw = {k: v for k, v in zip(("N", "M", "P"), a[:3]) if v > 0}
    if kw:
        cfg = I.scaled(cfg, **kw)
    reps = a[3] if len(a) > 3 else 3
    x, y, w = (torch.from_numpy(v).cuda() for v in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    par = I.kernel_param(cfg) if cfg.kind != "negdist" else 1.0
    ws = torch.empty(S.sks_workspace_size(cfg.N, cfg.M, cfg.d, cfg.kind, par, cfg.P), dtype=torch.uint8, device="cuda")
    out = torch.empty(cfg.M, device="cuda")
    S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, out=out, workspace=ws)
    S.sks_profile_enable(True)
    S.sks_profile_read()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, out=out, workspace=ws)
    ev[1].record()
    torch.cuda.synchronize()
    prof = {k: round(v[0] / reps, 4) for k, v in S.sks_profile_read().items() if v[1]}
    print(json.dumps({"config": name, "N": cfg.N, "M": cfg.M, "P": cfg.P, "ms": ev[0].elapsed_time(ev[1]) / reps,
                      "kernels_ms": prof, "plan": S.sks_last_plan()}))


if __name__ == "__main__":
    main()
