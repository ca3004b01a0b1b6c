"""Small invocations of every kernel of libsks for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the projection variants (TF32x2, FP16x2 with and without the rerun, BF16x3), the sort path (few and many owners),
the Fourier path (NFFT private / shared spreading, NDFT), the Laplacian combination, the fused large-N kernels,
sks_sum_1d, async + graph calls.  Sizes are cfg1-like except where a path needs more points.
    compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_08260_b200 as S  # noqa: E402
from paper_2401_08260_b200 import build  # noqa: E402


def main(big=True):
    build.build()
    rng = np.random.default_rng(0)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    runs = []
    for d, N, M, P, kind, scale, kw in [
        (3, 1000, 1000, 64, "gaussian", 1.0, {}),                      # cfg1
        (3, 1000, 1000, 64, "gaussian", 1.0, {"engine": "ndft"}),
        (50, 3000, 1000, 16, "negdist", 1.0, {}),                      # sort path, few owners
        (50, 2000, 500, 16, "laplacian", 2.0, {}),                     # sort + Fourier (shared-grid spread)
        (50, 2000, 500, 8, "matern", 4.0, {}),
        (52, 2000, 300, 8, "negdist", 1.0, {"projection": "bf16x3"}),
        (300, 700, 200, 8, "gaussian", 20.0, {}),                      # FP16x2
        (300, 700, 200, 8, "gaussian", 20.0, {"projection": "tf32x2"}),
        (257, 500, 100, 8, "negdist", 1.0, {}),                        # d % 4 != 0: BF16x3 split pass
    ]:
        x, y = rng.normal(size=(N, d)), rng.normal(size=(M, d))
        w = rng.uniform(-1, 1, N)
        s = S.sks_sum(dev(x), dev(y), dev(w), kind, scale, P, 7, **kw)
        runs.append((kind, d, float(s.abs().sum())))
    # FP16x2 range rerun (a point beyond the sampled scale)
    x = rng.normal(size=(700, 256)).astype(np.float32)
    x[1] *= 1e5
    S.sks_sum(dev(x), dev(rng.normal(size=(100, 256))), dev(rng.uniform(0, 1, 700)), "negdist", 1.0, 8, 3)
    # many owners (> 128 per slice: plan bases, global owner table) and sks_sum_1d
    zx = rng.normal(size=(1, 600000)).astype(np.float32)
    zy = rng.normal(size=(1, 300)).astype(np.float32)
    S.sks_sum_1d(dev(zx), dev(zy), dev(rng.uniform(0, 1, 600000)), 50, "negdist", 1.0)
    S.sks_sum_1d(dev(zx[:, :5000]), dev(zy), dev(rng.uniform(0, 1, 5000)), 10, "gaussian", 1.0)
    # async + graph
    x, y, w = dev(rng.normal(size=(1000, 3))), dev(rng.normal(size=(1000, 3))), dev(rng.uniform(-1, 1, 1000))
    ws = torch.empty(S.sks_workspace_size(1000, 1000, 3, "gaussian", 1.0, 64), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        S.sks_sum(x, y, w, "gaussian", 1.0, 64, 1, workspace=ws, graph=True)
    S.sks_sync_status(ws)
    if big:   # the fused large-N kernels (N >= 2^18)
        N = 300_000
        x = rng.normal(size=(N, 100)).astype(np.float32)
        S.sks_sum(dev(x), dev(rng.normal(size=(2000, 100))), dev(rng.uniform(-1, 1, N)), "gaussian", 15.0, 20, 5)
        assert S.sks_last_plan()["fused"] == 1
        # the fused spread's other footprint classes (<= 64 cells: 4 private copies; wider: one shared column with
        # shared-memory atomics) and an odd window width
        for kw in (dict(window_w=7), dict(oversample=4), dict(oversample=8), dict(window_w=5, oversample=8)):
            S.sks_sum(dev(x), dev(rng.normal(size=(2000, 100))), dev(rng.uniform(-1, 1, N)), "gaussian", 15.0, 20, 5,
                      **kw)
            assert S.sks_last_plan()["fused"] == 1
    torch.cuda.synchronize()
    print("sanitize run OK", runs)


if __name__ == "__main__":
    main(big="--no-big" not in sys.argv)
