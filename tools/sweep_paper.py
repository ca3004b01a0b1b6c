"""The paper's Sec. 4.1 / 4.2 experiment (Fig. 3) at B200 scale -- SURVEY.md §8(f) item f3.

Workload: x, y ~ N(0, 0.1^2 I), w ~ U[0,1], Gaussian sigma = 1, Matern nu = 3/2 beta = 1, negative
distance, Laplacian alpha = 0.5 (ell = 2).  Three sweeps, per kernel:
  time vs N   (d = 50, several P): the fast summation through the C-ABI (CUDA events) next to a naive O(NM)
              PyTorch brute force on the same GPU (cdist + kernel, chunked; only up to N = 1e5);
  error vs d  (N = 1e4, several P): per-summand error ||s_true - s_fast||_1 / (M sum|w|) against the
              exact d-dimensional sum, oracle (a), on a target subset;
  error vs P  (N = 1e4, several d): same error; the fitted log-log slope checks O(P^{-1/2}) (Prop. 2.6, Thm 2.7).

    python tools/sweep_paper.py [--quick] [--out profiles/r01_fig3]      (needs a GPU; writes .json and .md)
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2401_08260_b200 import inputs as I  # noqa: E402

KERNELS = [("gaussian", "paper_gauss"), ("matern", "paper_matern"), ("negdist", "paper_negdist"),
           ("laplacian", "paper_laplace")]


def naive_gpu(torch, x, y, w, kind, param, matern_p=1):
    """exact O(NM) sum on the GPU in fp32 (PyTorch cdist + kernel), the paper's naive comparison"""
    out = torch.empty(y.shape[0], dtype=torch.float64, device=y.device)
    for m0 in range(0, y.shape[0], 4096):
        r = torch.cdist(y[m0:m0 + 4096], x)
        if kind == "gaussian":
            k = torch.exp(-r * r / (2 * param * param))
        elif kind == "negdist":
            k = -r
        elif kind == "laplacian":
            k = torch.exp(-r / param)
        else:   # Matern nu = 3/2 (P:1163 with p = 1)
            a = math.sqrt(3.0) * r / param
            k = (1 + a) * torch.exp(-a)
        out[m0:m0 + 4096] = (k @ w).double()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="small grids (smoke)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_fig3"))
    args = ap.parse_args()
    import torch

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200 import build as B
    B.build()
    O.build()
    dev = torch.device("cuda", 0)
    recs = []

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    Ns = [1000, 10_000, 100_000] if args.quick else [1000, 10_000, 100_000, 1_000_000, 10_000_000]
    Ps_time = [64, 256] if args.quick else [64, 256, 1024]
    ds = [3, 50, 500] if args.quick else [3, 10, 50, 100, 500, 1000]
    Ps_err = [16, 64, 256] if args.quick else [16, 64, 256, 1024, 4096]
    n_tgt = 300

    for kind, cname in KERNELS:
        base = I.CONFIGS[cname]
        param = I.kernel_param(base)
        scale = param if kind != "negdist" else 1.0
        # ---- time vs N (d = 50)
        for N in Ns:
            cfg = I.scaled(base, N=N, M=N)
            x, y, w = (torch.from_numpy(a).to(dev) for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
            for P in Ps_time:
                ms = timed(lambda: S.sks_sum(x, y, w, kind, scale, P, cfg.dir_seed, matern_p=cfg.matern_p))
                recs.append({"sweep": "time_vs_N", "kernel": kind, "d": cfg.d, "N": N, "P": P, "ms": ms,
                             "engine": S.sks_last_plan()["engine"]})
                print(json.dumps(recs[-1]), flush=True)
            if N <= 100_000:
                ms = timed(lambda: naive_gpu(torch, x, y, w, kind, param, cfg.matern_p), reps=2)
                recs.append({"sweep": "time_vs_N", "kernel": kind, "d": cfg.d, "N": N, "P": None, "ms": ms,
                             "impl": "naive O(NM) PyTorch (cdist), fp32"})
                print(json.dumps(recs[-1]), flush=True)
            del x, y, w
            torch.cuda.empty_cache()
        # ---- error vs d and vs P (N = 1e4)
        for d in sorted(set(ds) | {10, 50, 500}):
            cfg = dataclasses.replace(base, d=d)
            xn, yn, wn = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
            tgt = I.target_subset(cfg.M, n_tgt)
            try:
                exact = O.exact_sum(kind, param if kind != "negdist" else 0.0, xn, yn[tgt], wn, matern_p=cfg.matern_p)
            except Exception as e:   # the oracle refuses a conditioning it cannot vouch for
                print(f"skip {kind} d={d}: {e}", flush=True)
                continue
            x, y, w = (torch.from_numpy(a).to(dev) for a in (xn, yn, wn))
            sw = float(np.abs(wn.astype(np.float64)).sum())
            Pset = sorted(set(Ps_err if d in (10, 50, 500) else []) | set(Ps_time if d in ds else []))
            for P in Pset:
                s = S.sks_sum(x, y, w, kind, scale, P, cfg.dir_seed, matern_p=cfg.matern_p).cpu().numpy()
                diff = s[tgt].astype(np.float64) - exact
                recs.append({"sweep": "error", "kernel": kind, "d": d, "N": cfg.N, "P": P,
                             "per_summand": float(np.abs(diff).sum() / (len(tgt) * sw)),
                             "max_over_sumw": float(np.abs(diff).max() / sw)})
                print(json.dumps(recs[-1]), flush=True)
    json.dump(recs, open(args.out + ".json", "w"), indent=0)

    # ---- markdown summary
    lines = ["# Paper Fig. 3 workload at B200 scale (tools/sweep_paper.py)", "",
             "x, y ~ N(0, 0.1^2 I), w ~ U[0,1] (P:666-667); Gaussian sigma=1, Matern nu=3/2 beta=1, negative distance,",
             "Laplacian alpha=0.5.  Times: CUDA events around sks_sum (inputs resident on the GPU).  Errors: per-summand",
             "||s_true - s_fast||_1 / (M sum|w|) (P:677) on 300 targets against the exact sum (oracle (a)).", ""]
    for kind, _ in KERNELS:
        lines += [f"## {kind}", "", "| N | " + " | ".join(f"P={P} ms" for P in Ps_time) + " | naive ms |",
                  "|---" * (len(Ps_time) + 2) + "|"]
        for N in Ns:
            row = [f"{N:.0e}"]
            for P in Ps_time:
                r = [x for x in recs if x["sweep"] == "time_vs_N" and x["kernel"] == kind and x["N"] == N and x["P"] == P]
                row.append(f"{r[0]['ms']:.3f}" if r else "-")
            r = [x for x in recs if x["sweep"] == "time_vs_N" and x["kernel"] == kind and x["N"] == N and x["P"] is None]
            row.append(f"{r[0]['ms']:.2f}" if r else "-")
            lines.append("| " + " | ".join(row) + " |")
        errs = [x for x in recs if x["sweep"] == "error" and x["kernel"] == kind]
        dset = sorted({x["d"] for x in errs})
        Pall = sorted({x["P"] for x in errs})
        lines += ["", "| d | " + " | ".join(f"P={P}" for P in Pall) + " | slope vs P |", "|---" * (len(Pall) + 2) + "|"]
        for d in dset:
            row, pts = [str(d)], []
            for P in Pall:
                r = [x for x in errs if x["d"] == d and x["P"] == P]
                row.append(f"{r[0]['per_summand']:.2e}" if r else "-")
                if r and r[0]["per_summand"] > 0:
                    pts.append((math.log(P), math.log(r[0]["per_summand"])))
            slope = np.polyfit(*zip(*pts), 1)[0] if len(pts) >= 3 else float("nan")
            row.append(f"{slope:.2f}" if len(pts) >= 3 else "-")
            lines.append("| " + " | ".join(row) + " |")
        lines.append("")
    open(args.out + ".md", "w").write("\n".join(lines))
    print("wrote", args.out + ".json", args.out + ".md")


if __name__ == "__main__":
    main()
