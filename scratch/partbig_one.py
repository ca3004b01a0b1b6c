import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
dev = torch.device("cuda", 0)
N = 10_000_000
g = torch.Generator(device=dev); g.manual_seed(5)
x = 0.1 * torch.randn(N, 100, device=dev, generator=g); y = 0.1 * torch.randn(N, 100, device=dev, generator=g)
w = torch.rand(N, device=dev, generator=g)
S.sks_sum(x, y, w, "negdist", 1.0, 16, 7); torch.cuda.synchronize()
print("ok")
