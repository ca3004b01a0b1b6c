import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_08260_b200 as S
dev = torch.device("cuda", 0)
for N in (100_000, 1_000_000, 3_000_000, 10_000_000):
    g = torch.Generator(device=dev); g.manual_seed(5)
    x = 0.1 * torch.randn(N, 100, device=dev, generator=g); y = 0.1 * torch.randn(N, 100, device=dev, generator=g)
    w = torch.rand(N, device=dev, generator=g)
    P = 100
    f = lambda: S.sks_sum(x, y, w, "negdist", 1.0, P, 7)
    f(); torch.cuda.synchronize()
    S.sks_profile_enable(True); S.sks_profile_read()
    f(); torch.cuda.synchronize()
    prof = {k: round(v[0], 3) for k, v in S.sks_profile_read().items() if v[1]}
    S.sks_profile_enable(False)
    print(json.dumps({"N": N, "prof": prof, "plan": {k: S.sks_last_plan()[k] for k in ("slice_batch", "n_batches")}}), flush=True)
    del x, y, w; torch.cuda.empty_cache()
