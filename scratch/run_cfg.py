"""run sks_sum on a (scaled) config a few times (for ncu captures)"""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
from paper_2401_08260_b200 import inputs as I
name = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 0; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = I.CONFIGS[name]
if N: cfg = I.scaled(cfg, N=N, M=N)
dev = torch.device("cuda", 0)
x, y, w = (torch.from_numpy(a).to(dev) for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
par = I.kernel_param(cfg)
for _ in range(reps):
    s = S.sks_sum(x, y, w, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p)
torch.cuda.synchronize()
print(S.sks_last_plan())
