"""The paper's GPU benchmark (Table 3; RTX 4090, PyTorch) at B200 scale -- the slicing rows.

Workload (P:966-969 -> P:666-667): d = 100, M = N, x, y ~ N(0, 0.1^2 I), w ~ U[0, 1], Gaussian sigma^2 = 1
(the paper's 1D engine: NDFT; here the NFFT default and the NDFT engine) and the negative distance
kernel (sorting).  N in {1e4, 1e5, 1e6, 1e7}, P in {100, 1000, 2000, 5000}.  Times: CUDA events around
sks_sum with the inputs resident on the GPU (the paper reports wall-clock seconds of its PyTorch code); the
paper's numbers are copied from BASELINE.md (context, another GPU).

    python tools/table3.py [--out profiles/r01_table3] [--quick]        (needs a GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# seconds on one RTX 4090, rows P, columns N
PAPER = {
    "gaussian": {100: [0.0065, 0.014, 0.279, 2.72], 1000: [0.0493, 0.144, 2.80, 25.4],
                 2000: [0.0953, 0.283, 5.70, 50.9], 5000: [0.2365, 0.713, 13.1, 127.2]},
    "negdist": {100: [0.0021, 0.009, 0.070, 1.51], 1000: [0.0092, 0.093, 0.686, 15.1],
                2000: [0.0192, 0.183, 1.37, 30.17], 5000: [0.0455, 0.456, 3.42, 75.58]},
}
NS = [10_000, 100_000, 1_000_000, 10_000_000]
PS = [100, 1000, 2000, 5000]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_table3"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200 import build as B
    B.build()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    recs = []
    Ns = NS[:2] if args.quick else NS
    for j, N in enumerate(Ns):
        g.manual_seed(2401 + N)
        x = 0.1 * torch.randn(N, 100, device=dev, generator=g)
        y = 0.1 * torch.randn(N, 100, device=dev, generator=g)
        w = torch.rand(N, device=dev, generator=g)
        for kind, engine in [("gaussian", "nfft"), ("gaussian", "ndft"), ("negdist", "auto")]:
            for P in PS:
                ws = torch.empty(S.sks_workspace_size(N, N, 100, kind, 1.0, P, 0, P, engine=engine),
                                 dtype=torch.uint8, device=dev)
                f = lambda: S.sks_sum(x, y, w, kind, 1.0, P, 7, workspace=ws, engine=engine)  # noqa: E731
                try:
                    f()
                except Exception as e:   # e.g. the NDFT engine refuses bands wider than 32 coefficients
                    recs.append({"kernel": kind, "engine": engine, "N": N, "P": P, "error": str(e)})
                    print(json.dumps(recs[-1]), flush=True)
                    continue
                reps = max(1, min(20, int(2e9 // (N * P))))   # short calls: more repetitions
                for _ in range(min(reps, 3)):   # warm-up (clocks, caches) before the timed calls
                    f()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    f()
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / reps
                paper_s = PAPER[kind][P][j]
                recs.append({"kernel": kind, "engine": S.sks_last_plan()["engine"], "N": N, "P": P, "ms": ms,
                             "slice_points_per_s": 2 * N * P / (ms * 1e-3), "paper_s_rtx4090": paper_s,
                             "ratio_vs_paper": paper_s * 1e3 / ms})
                print(json.dumps(recs[-1]), flush=True)
                del ws
                torch.cuda.empty_cache()
        del x, y, w
        torch.cuda.empty_cache()
    json.dump(recs, open(args.out + ".json", "w"), indent=0)
    lines = ["# The paper's Table 3 (GPU, slicing rows) at B200 scale (tools/table3.py)", "",
             "d = 100, M = N, x, y ~ N(0, 0.1^2 I), w ~ U[0,1] (P:966-969, P:666-667).  B200: CUDA events around",
             "`sks_sum`, inputs resident on the GPU.  Paper: wall-clock seconds on one RTX 4090 (BASELINE.md, P:929-954;",
             "context from another GPU, not a target).  Each cell: B200 ms (paper ms, ratio paper / B200).", ""]
    for kind, engine in [("gaussian", 1), ("gaussian", 2), ("negdist", 0)]:
        title = {1: "Gaussian sigma^2 = 1, NFFT", 2: "Gaussian sigma^2 = 1, NDFT (the paper's engine)",
                 0: "Negative distance (sorting)"}[engine]
        lines += [f"## {title}", "", "| P \\ N | " + " | ".join(f"{n:.0e}" for n in Ns) + " |",
                  "|---" * (len(Ns) + 1) + "|"]
        for P in PS:
            row = [str(P)]
            for N in Ns:
                r = [q for q in recs if q["kernel"] == kind and q.get("engine") == engine and q["N"] == N
                     and q["P"] == P and "ms" in q]
                row.append(f"{r[0]['ms']:.3g} ({1e3 * r[0]['paper_s_rtx4090']:.3g}, x{r[0]['ratio_vs_paper']:.0f})"
                           if r else "-")
            lines.append("| " + " | ".join(row) + " |")
        lines.append("")
    open(args.out + ".md", "w").write("\n".join(lines))
    print("wrote", args.out + ".json", args.out + ".md")


if __name__ == "__main__":
    main()
