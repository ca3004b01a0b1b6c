"""A/B of the NFFT window (taps w, oversampling os) on one configuration: device time per call at full size
and the error against the CPU oracle on a scaled-down copy of the same workload (the window error does not depend
on N).    python tools/window_ab.py cfg5 "6,2 5,2 5,4 4,4" [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2401_08260_b200 as S  # noqa: E402
from paper_2401_08260_b200 import build, inputs as I  # noqa: E402


def dev(cfg):
    return tuple(torch.from_numpy(v).cuda() for v in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))


def main():
    build.build()
    O.build()
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    combos = [tuple(int(v) for v in c.split(",")) for c in (sys.argv[2] if len(sys.argv) > 2 else "6,2 5,4").split()]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    full = I.CONFIGS[name]
    small = I.scaled(full, N=300001, M=2000, P=16)   # N >= 2^18: the fused path
    par = I.kernel_param(full)
    xs, ys, ws_ = I.points(small, "x"), I.points(small, "y"), I.weights(small)
    tgt = I.target_subset(small.M, 16)
    ref = O.sliced_sum(small.kind, par, xs, ys, ws_, small.P, small.dir_seed, targets=tgt, matern_p=small.matern_p)
    sw = np.abs(ws_.astype(np.float64)).sum()
    dsm = tuple(torch.from_numpy(v).cuda() for v in (xs, ys, ws_))
    # diagnostic only: a wide window's result on all targets (the A/B's common yardstick beside the oracle sample)
    wide = S.sks_sum(*dsm, small.kind, par, small.P, small.dir_seed, matern_p=small.matern_p, window_w=10,
                     oversample=2).cpu().numpy()
    x, y, w = dev(full)
    out = torch.empty(full.M, device="cuda")
    for (ww, os_) in combos:
        kw = dict(window_w=ww, oversample=os_)
        rec = {"w": ww, "os": os_}
        try:
            s = S.sks_sum(*dsm, small.kind, par, small.P, small.dir_seed, matern_p=small.matern_p, **kw).cpu().numpy()
            rec["err"] = float(np.max(np.abs(s[tgt] - ref)) / sw)
            rec["vs_w10"] = float(np.max(np.abs(s - wide)) / sw)
            rec["small_fused"] = S.sks_last_plan()["fused"]
        except Exception as e:  # noqa: BLE001
            rec["err"] = str(e)[:80]
        try:
            wsz = S.sks_workspace_size(full.N, full.M, full.d, full.kind, par, full.P, **kw)
            wk = torch.empty(wsz, dtype=torch.uint8, device="cuda")
            S.sks_sum(x, y, w, full.kind, par, full.P, full.dir_seed, out=out, workspace=wk, **kw)
            S.sks_profile_enable(True)
            S.sks_profile_read()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(reps):
                S.sks_sum(x, y, w, full.kind, par, full.P, full.dir_seed, out=out, workspace=wk, **kw)
            ev[1].record()
            torch.cuda.synchronize()
            rec["ms"] = ev[0].elapsed_time(ev[1]) / reps
            rec["kernels_ms"] = {k: round(v[0] / reps, 3) for k, v in S.sks_profile_read().items() if v[1]}
            rec["plan"] = S.sks_last_plan()
            S.sks_profile_enable(False)
            del wk
        except Exception as e:  # noqa: BLE001
            rec["full"] = str(e)[:200]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
