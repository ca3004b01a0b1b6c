import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
import oracle as O
for n, d, P in [(1000, 50, 70), (3000, 100, 64), (300, 3, 64)]:
    rng = np.random.default_rng(n + d)
    pts = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    z = S.sks_project(torch.from_numpy(pts).cuda(), P, seed=7).cpu().numpy()
    zo = O.project(pts, O.unit_directions(P, d, 7))
    scale = np.linalg.norm(pts.astype(np.float64), axis=1).max()
    print(n, d, P, "max err / scale", np.max(np.abs(z - zo)) / scale)
