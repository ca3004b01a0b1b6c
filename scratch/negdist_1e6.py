import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
dev = torch.device("cuda", 0)
for N in (1_000_000, 10_000_000):
    g = torch.Generator(device=dev); g.manual_seed(2401 + N)
    x = 0.1 * torch.randn(N, 100, device=dev, generator=g); y = 0.1 * torch.randn(N, 100, device=dev, generator=g)
    w = torch.rand(N, device=dev, generator=g)
    for P in (100, 1000):
        f = lambda: S.sks_sum(x, y, w, "negdist", 1.0, P, 7)
        f(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        a.record()
        for _ in range(reps): f()
        b.record(); torch.cuda.synchronize()
        print(json.dumps({"N": N, "P": P, "ms": a.elapsed_time(b) / reps}), flush=True)
    del x, y, w; torch.cuda.empty_cache()
