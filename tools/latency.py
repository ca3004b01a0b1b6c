"""Per-call latency of small problems (BASELINE configs[0] = cfg1 by default): eager calls (synchronous status
read), async calls, and CUDA-graph replays (sks_options.graph), timed with CUDA events over many back-to-back
calls on one stream.  SURVEY Sec. 7 hard part 9: cfg1 is launch-latency bound (target 10-30 us)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_08260_b200 as S  # noqa: E402
from paper_2401_08260_b200 import build, inputs as I  # noqa: E402


def main(name="cfg1", iters=200):
    build.build()
    cfg = I.CONFIGS[name]
    x, y, w = (torch.from_numpy(a).cuda() for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    par = I.kernel_param(cfg) if cfg.kind != "negdist" else 1.0
    ws = torch.empty(S.sks_workspace_size(cfg.N, cfg.M, cfg.d, cfg.kind, par, cfg.P), dtype=torch.uint8, device="cuda")
    out = torch.empty(cfg.M, device="cuda")
    res = {"config": name}
    for mode, kw in [("sync", {}), ("async", {"async_": True}), ("graph", {"graph": True})]:
        for _ in range(5):
            S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, out=out, workspace=ws, **kw)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, out=out, workspace=ws, **kw)
        b.record()
        torch.cuda.synchronize()
        if mode != "sync":
            S.sks_sync_status(ws)
        res[mode + "_us_per_call"] = a.elapsed_time(b) * 1e3 / iters
    res["plan"] = S.sks_last_plan()
    print(json.dumps(res))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["cfg1"]))
