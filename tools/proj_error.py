"""Projection error (row a1) per variant and dimension against the fp64 oracle, in units of max ||pt||, plus the
signed mean relative error (a systematic shrink shows the tensor core's truncating fp32 accumulation)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, paper_2401_08260_b200 as S
from paper_2401_08260_b200 import build
build.build()
for mode in ["tf32x2", "fp16x2", "bf16x3"]:
    for n, d, P in [(300, 3, 64), (1000, 50, 70), (700, 100, 300), (257, 784, 33), (257, 1536, 17), (129, 3072, 17)]:
        pts = np.random.default_rng(n + d).uniform(-1, 1, (n, d)).astype(np.float32)
        z = S.sks_project(torch.from_numpy(pts).cuda(), P, seed=7, projection=mode).cpu().numpy().astype(np.float64)
        zo = O.project(pts, O.unit_directions(P, d, 7))
        scale = np.linalg.norm(pts.astype(np.float64), axis=1).max()
        big = np.abs(zo) > 0.1 * np.abs(zo).max()
        shrink = np.mean((np.abs(z[big]) - np.abs(zo[big])) / np.abs(zo[big]))
        print(f"{mode:7s} d={d:5d}: max|dz|/||pt|| = {np.max(np.abs(z - zo)) / scale:.3e}   mean rel (|z|-|zo|)/|zo| = {shrink:+.3e}")
