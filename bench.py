#!/usr/bin/env python
"""bench.py -- throughput of the sliced fast kernel summation hot path (Alg. 1) on B200.

Metric (BASELINE.json): slice-points/s = (N+M)*P / t and ms per kernel sum.  A "step" is one full
kernel sum (all Sec. 8a rows: projection, sort/Fourier 1D engines, slice mean, and for N>1 GPUs the
NCCL all-reduce of the M-length partial sums) over one batch of seeded synthetic inputs already
resident in HBM.  Default workload: BASELINE.json configs[4] ("cfg5", Gaussian, d=100, N=M=1e7, P=512), the
largest configuration that fits one GPU (all 512 slices on one GPU at N=1; 64 per GPU at N=8) and the one the
1 -> 8 GPU target is defined on.  Slices are partitioned over ranks ([rP/G, (r+1)P/G)) by
parallel.distributed_sliced_sum, whose one NCCL all-reduce combines the partial sums; scaling is strong (the
total work is fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the launch stream,
L2 flushed (256 MiB write) before every step outside the events; barrier + synchronize around the
timed region; max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2401_08260_b200 import inputs as I  # noqa: E402

METRIC = "slice-points/s ((N+M)·P) and ms per kernel sum at 1/2/4/8 B200"
UNIT = "slice-points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg5", choices=sorted(I.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="async", choices=["sync", "async", "graph"],
                    help="sks_options for the device-resident step: sync (status read per call), async (no host "
                         "synchronisation; status read after the timed region), graph (async + CUDA-graph replay)")
    ap.add_argument("--shard", default="auto", choices=["auto", "slices", "points"],
                    help="N > 1: slice ranges + one all-reduce of the sums, or point rows + the in-call exchanges of "
                         "the large-N Fourier path (parallel.point_sharded_sum); auto = points where that path runs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# ------------------------------------------------------------------ roofline model per kernel
# Algorithmic work per SLICE-POINT (one point of L = N + M on one slice), SURVEY.md Sec. 8(d) / DESIGN.md Sec. 6:
#   projection  2 d fp32-accurate flops + 4 B projection store (+ 4 d / P_local B of input)
#   sort path   84 B: 4 B projection store (counted in the projection) + 80 B for the sort stage (4 LSD passes x
#               (4 B key + 4 B payload) x read/write = 64 B, 4 B histogram, 8 B scan read, ~4 B output)
#   Fourier     4 B projection load (+ 2m window taps of arithmetic; spread over the x, interpolation over the y)
# The "compulsory" figures are this build's own minimum traffic (each input read once, each output written
# once: the owner-partitioned sort moves 28 B per slice-point, not 80), reported beside the Sec. 8(d) fraction.
SORT_B_PER_SP = 80.0


def roofline_model(slot, cfg, P, plan):
    """(Sec. 8(d) bytes, compulsory bytes, (bound kind, algorithmic flops)) of ONE launch of a kernel slot over P
    slices."""
    N, M, d = cfg.N, cfg.M, cfg.d
    L = N + M
    n = plan.get("n_grid", 0) or 0
    w = plan.get("window_w", 6) or 6
    if slot == "project":
        by = 4 * L * d + 4 * L * P
        return by, by, ("tensor", 2.0 * L * d * P)
    if slot == "split3":
        return 4 * L * d, 4 * L * d + 6 * L * ((d + 63) // 64 * 64), None
    comp = {"sp_hist": 4 * L * P, "sp_part": 4 * L * P + 4 * N + (8 * N + 8 * M) * P,
            "sp_owner": (8 * N + 8 * M) * P, "sp_gather": 8 * M * P + 16 * M}
    if slot in comp:
        return comp[slot], comp[slot], None
    if slot == "sortsum":   # the sort stage (fork .. join of its kernels on two streams)
        return SORT_B_PER_SP * L * P, sum(comp.values()), None
    if plan.get("fused"):   # the fused large-N path (fused.cu): projection + spread / projection + interpolation
        dp16 = (d + 7) // 8 * 8
        if slot == "minmax":   # source prep: one pass over x and y (norm bounds) writing their fp16 hi / lo rows
            by = 4 * (N + M) * d + 4 * (N + M) * dp16 + 8 * N
            return by, by, None
        if slot == "spread":   # per x slice-point: 2 d projection flops (tensor) + w taps (FP32); x's fp16 hi / lo
            by = 4 * N * dp16 + 4 * N + 4 * n * P
            return by, by, ("tensor", 2.0 * N * d * P), ("alu", 2.0 * N * P * w * 5)
        if slot == "eval":     # per y slice-point: 2 d projection flops (tensor) + one degree-7 Horner (FP32)
            by = 4 * M * dp16 + 8 * M + 4 * n * P
            return by, by, ("tensor", 2.0 * M * d * P), ("alu", 2.0 * M * P * 7)
    if slot == "spread":    # per x slice-point: w taps, each a degree-7 window polynomial (even/odd form: 4 FMA
        #                     per tap) and one FMA into the grid
        return 4 * N * P, 4 * N * P + 4 * N + 4 * n * P, ("alu", 2.0 * N * P * w * 5)
    if slot == "eval":      # per y slice-point: one degree-7 Horner (7 FMA) on the cell's interpolation polynomial
        return 4 * M * P, 4 * M * P + 16 * M + 4 * n * P, ("alu", 2.0 * M * P * 7)
    if slot == "fft_filter":
        return 8 * n * P, 8 * n * P + 4 * (n // 2 + 1) * P, None
    if slot == "plan_D":
        return 4 * (n // 2 + 1) * P, 4 * (n // 2 + 1) * P, None
    return 0, 0, None


def tensor_peak(pk, pmode):
    """fp32-accurate flops/s of the projection (reading R2): TF32x2 = two tf32 MMAs per product at half the bf16
    rate (the guide's nominal tf32:bf16 ratio), FP16x2 = two fp16 MMAs at the bf16 rate, BF16x3 = three."""
    div = {3: 4.0, 4: 2.0}.get(pmode, 3.0)
    src = {3: "MEASURED_PEAKS.json bf16_tflops / 4 (TF32x2: 2 tf32 MMAs per fp32 product, tf32 = bf16 / 2 nominal)",
           4: "MEASURED_PEAKS.json bf16_tflops / 2 (FP16x2: 2 fp16 MMAs per fp32 product, fp16 = bf16 rate)"}
    return pk["bf16_tflops"] / div, src.get(pmode, "MEASURED_PEAKS.json bf16_tflops / 3 (BF16x3)")


def alu_peak(pk):
    """FP32 FMA peak (TFLOP/s, source): the measured packed-FMA (FFMA2, the fused spread's form) throughput of a B200
    at its maximum clock (tools/fp32_peak.cu -> profiles/r02/fp32_peak.json: 74.3 TF/s, scalar 3-register FFMA 72.5),
    else the unit counts (148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz, B200_PROFILING.md)"""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "fp32_peak.json")) as f:
            m = json.load(f)
        return (float(m["ffma2_tflops"]), "measured FFMA2 throughput at %d MHz (tools/fp32_peak.cu, "
                "profiles/r02/fp32_peak.json)" % m["max_clock_mhz"])
    except (OSError, KeyError, ValueError):
        return (148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
                "148 SMs x 128 FP32 lanes x 2 flop/FMA x sm_max_mhz (B200_PROFILING unit counts)")


# the kernels of a bench slot as they appear in the committed ncu summaries (tools/ncu_summary.py)
NCU_KERNELS = {"spread": ("k_proj_spread", "k_spread"), "eval": ("k_proj_eval", "k_eval"),
               "project": ("k_proj_pair", "k_proj_tc"), "minmax": ("k_prep_f16",)}


def ncu_context(cfg_name, slot):
    """Context for the roofline record, not a measurement of this run: the pipe utilisations of the slot's kernel
    in the committed ncu --set full summary of this configuration (profiles/r02/ncu_<cfg>*.csv), where one exists
    -- the shared-memory data pipe (LSU + tensor-core operand wavefronts), tensor pipe, issue slots."""
    import csv
    import glob
    names = NCU_KERNELS.get(slot, ())
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02", f"ncu_{cfg_name}*.csv"))):
        try:
            rows = list(csv.DictReader(open(path)))
        except OSError:
            continue
        for n in names:
            for r in rows:
                if n in r.get("kernel", ""):
                    f = lambda k: float(r[k]) if r.get(k) not in (None, "") else None
                    lsu, tc = f("smem_lsu_wavefronts_pct"), f("smem_tc_wavefronts_pct")
                    return {"source": os.path.relpath(path, ROOT), "kernel": r["kernel"],
                            "smem_pipe_pct": (lsu or 0.0) + (tc or 0.0) if lsu is not None else None,
                            "tensor_pipe_active_pct": f("tensor_pipe_active_pct"),
                            "issue_active_pct": f("issue_active_pct"), "fma_pipe_pct": f("fma_pipe_pct")}
    return None


def roofline(slot, cfg, P, plan, ms_per_launch, pk, traffic):
    """achieved / peak of one kernel, Sec. 8(d) units: the bound is the larger of the HBM time of its Sec. 8(d)
    bytes and the time of its algorithmic arithmetic at peak (tensor for the projection, FP32 FMA for the
    spread / interpolation).  Also the compulsory-traffic fraction (this build's own minimum bytes)."""
    by, comp, *work = roofline_model(slot, cfg, P, plan)
    work = [x for x in work if x]
    t = ms_per_launch * 1e-3
    peaks_tf = {"tensor": tensor_peak(pk, plan.get("proj_mode")), "alu": alu_peak(pk)}
    hbm = pk["hbm_gbs"]
    # the binding resource of the model: the largest of the HBM time and each arithmetic unit's time at its peak
    kind, fl = max(work, key=lambda kf: kf[1] / (peaks_tf[kf[0]][0] * 1e12)) if work else (None, 0.0)
    if fl and fl / (peaks_tf[kind][0] * 1e12) > by / (hbm * 1e9):
        r = {"kernel": slot, "bound": kind, "achieved": fl / t / 1e12, "peak": peaks_tf[kind][0], "unit": "TFLOP/s",
             "peak_source": peaks_tf[kind][1], "algorithmic_flops_per_launch": fl}
    else:
        r = {"kernel": slot, "bound": "hbm", "achieved": by / t / 1e9, "peak": hbm, "unit": "GB/s",
             "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else "")}
    r["frac"] = r["achieved"] / r["peak"]
    # every modelled resource's time at its peak / the launch time (the headline frac is the largest)
    r["frac_by_resource"] = {"hbm": by / (hbm * 1e9) / t,
                             **{k: f / (peaks_tf[k][0] * 1e12) / t for k, f in work}}
    r["model"] = "SURVEY.md Sec. 8(d) per-slice-point work x slice-points per launch"
    r["algorithmic_bytes_per_launch"] = by
    r["compulsory_bytes_per_launch"] = comp
    r["compulsory_frac"] = comp / t / 1e9 / hbm
    r["traffic"] = traffic
    return r


class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, dev_index):
        self.dev = dev_index
        self.proc = None
        self.path = os.path.join("/tmp", f"sks_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def rows(self):
        try:
            return sum(1 for r in open(self.path) if r.strip())
        except OSError:
            return 0

    def wait_rows(self, n, timeout_s):
        """block until the sampler has written at least n rows (short timed regions: nvidia-smi needs ~0.1-1 s
        to start, so the region is bracketed by samples taken just before and just after it)"""
        t0 = time.perf_counter()
        while self.proc is not None and self.rows() < n and time.perf_counter() - t0 < timeout_s:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        rows = [r for r in rows if len(r) == len(self.FIELDS)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle (CPU) timing
def oracle_sample(cfg, param, x, y, w, target_seconds):
    """time oracle (b) on a bounded sample of the workload; returns (slice-points/s extrapolated, cores, desc)."""
    import oracle as O
    kind_param = param if cfg.kind != "negdist" else 0.0
    P = cfg.P
    p_sub = P if cfg.N * cfg.d < 5e7 else max(1, P // 32)
    m = 4
    t = 0.0
    while True:
        tgt = I.target_subset(cfg.M, m, seed=777)
        t0 = time.perf_counter()
        O.sliced_sum(cfg.kind, kind_param, x, y, w, P, cfg.dir_seed, targets=tgt, p0=0, p1=p_sub, matern_p=cfg.matern_p)
        t = time.perf_counter() - t0
        if t >= target_seconds / 3 or m >= cfg.M:
            break
        m = min(cfg.M, max(m * 2, int(m * target_seconds / max(t, 1e-3) / 2)))
    frac = (len(tgt) / cfg.M) * (p_sub / P)
    value = (cfg.N + cfg.M) * P / (t / frac)
    desc = (f"oracle (b) on {len(tgt)} of {cfg.M} targets x {p_sub} of {P} slices x all {cfg.N} sources "
            f"({t:.2f} s); time extrapolated linearly in targets and slices")
    return value, O.num_threads(), desc, t


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    O.build()
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    param = I.kernel_param(cfg)
    kind_param = param if cfg.kind != "negdist" else 0.0
    P = cfg.P
    p_sub = P if cfg.N * cfg.d < 5e7 else max(1, P // 32)
    n_tgt = 8
    tgt = I.target_subset(cfg.M, n_tgt, seed=778)
    for _ in range(args.warmup):
        O.sliced_sum(cfg.kind, kind_param, x, y, w, P, cfg.dir_seed, targets=tgt[:2], p0=0, p1=1)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.sliced_sum(cfg.kind, kind_param, x, y, w, P, cfg.dir_seed, targets=tgt, p0=0, p1=p_sub,
                     matern_p=cfg.matern_p)
        ts.append(time.perf_counter() - t0)
    frac = (len(tgt) / cfg.M) * (p_sub / P)
    t_full = statistics.mean(ts) / frac
    value = (cfg.N + cfg.M) * P / t_full
    sample = (f"oracle (b) on {len(tgt)} of {cfg.M} targets x {p_sub} of {P} slices x all {cfg.N} sources per step; "
              f"time extrapolated linearly in targets and slices")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, param, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, param, G, points=False):
    return {"workload": cfg.name, "kernel": cfg.kind, "kernel_param": param, "d": cfg.d, "N": cfg.N, "M": cfg.M,
            "P": cfg.P, "slices_per_gpu": cfg.P if points else cfg.P // G,
            "parallelism": f"points{G}" if points else f"slices{G}",
            "l2": "flushed before every step (256 MiB write, outside the timed events)"}


def shard_by_points(shard, cfg, G):
    """the point-sharded large-N Fourier path (include/sks.h sks_exchange_fn) applies: every rank's share of the
    sources takes the fused path (api.cpp fused_shape)"""
    ok = cfg.kind in ("gaussian", "matern") and cfg.N // G >= (1 << 18) and cfg.d <= 128 and cfg.d % 4 == 0
    if shard == "points" and not ok:
        raise SystemExit(f"--shard points: {cfg.name} on {G} GPUs does not take the fused large-N Fourier path")
    return G > 1 and ok and shard != "slices"


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    cfg = I.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200 import build as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    G = world
    if world > 1:
        # NCCL init logging (stderr): the communicator lines show nranks / the NVLink(S) transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    S._lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())

    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    param = I.kernel_param(cfg)
    scale = param if cfg.kind != "negdist" else 1.0
    from paper_2401_08260_b200.parallel import make_exchange, point_range, slice_range
    points = shard_by_points(args.shard, cfg, G)
    if points and args.mode == "graph":
        raise SystemExit("--mode graph cannot replay the point-sharded call's exchanges")
    full = cfg
    if points:   # this rank's rows of x, w and y, all slices
        (n0, n1), (m0, m1) = point_range(rank, G, cfg.N), point_range(rank, G, cfg.M)
        x, y, w = (np.ascontiguousarray(a) for a in (x[n0:n1], y[m0:m1], w[n0:n1]))
        cfg = I.scaled(cfg, N=n1 - n0, M=m1 - m0)
        p0, p1 = 0, cfg.P
    else:
        p0, p1 = slice_range(rank, G, cfg.P)
    xd, yd, wd = (torch.from_numpy(a).to(dev) for a in (x, y, w))
    ws = torch.empty(S.sks_workspace_size(cfg.N, cfg.M, cfg.d, cfg.kind, scale, cfg.P, p0, p1, cfg.matern_p),
                     dtype=torch.uint8, device=dev)
    s = torch.empty(cfg.M, dtype=torch.float32, device=dev)
    if points:
        xfn, xerr = make_exchange(ws)
        counts = [point_range(r, G, full.M) for r in range(G)]
        s_parts = [torch.empty(b - a, dtype=torch.float32, device=dev) for a, b in counts]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    from paper_2401_08260_b200.parallel import distributed_sliced_sum

    mode_kw = {"sync": {}, "async": {"async_": True}, "graph": {"graph": True}}[args.mode]

    def step_slices(kw):   # this rank's slice range through the C-ABI, then the one all-reduce (SUM) of the partials
        distributed_sliced_sum(lambda a, b: S.sks_sum(xd, yd, wd, cfg.kind, scale, cfg.P, cfg.dir_seed, a, b,
                                                      cfg.matern_p, out=s, workspace=ws, **kw), cfg.P)

    def step_points(kw):   # this rank's point rows, all slices (three small exchanges inside the call), then the
        #                    all-gather that leaves the full result on every rank, as the slice mode does
        S.sks_sum(xd, yd, wd, cfg.kind, scale, cfg.P, cfg.dir_seed, 0, cfg.P, cfg.matern_p, out=s, workspace=ws,
                  exchange=xfn, **kw)
        dist.all_gather(s_parts, s)

    def step():
        (step_points if points else step_slices)(mode_kw)

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    plan = S.sks_last_plan()
    S.sks_profile_enable(True)
    S.sks_profile_read()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks.wait_rows(1, 5.0)
    r0 = clocks.rows()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    clocks.wait_rows(r0 + 1, 1.0)
    clk = clocks.stop()
    if args.mode != "sync":
        S.sks_sync_status(ws)   # the device status of the timed calls (raises on a failed call)
    kernels_from = "the timed region (CUDA events around every launch scope, on the launching stream)"
    if args.mode == "graph":
        # graph replays carry no per-launch events: the kernel breakdown comes from the same steps without the graph
        S.sks_profile_read()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            step_slices({"async_": True})
        torch.cuda.synchronize()
        S.sks_sync_status(ws)
        kernels_from = "an async (non-graph) pass of the same steps right after the timed graph region"
    prof = S.sks_profile_read()
    S.sks_profile_enable(False)
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = (full.N + full.M) * full.P / (ms * 1e-3)

    # ---- end to end through the public host-buffer API (H2D inputs + D2H result inside the timed region)
    e2e = None
    if not args.no_e2e:
        xh, yh, wh = (torch.from_numpy(a).pin_memory() for a in (x, y, w))
        sh = torch.empty(cfg.M, dtype=torch.float32).pin_memory()
        wsh = torch.empty(S.sks_workspace_size_host(cfg.N, cfg.M, cfg.d, cfg.kind, scale, cfg.P, p0, p1, cfg.matern_p),
                          dtype=torch.uint8, device=dev)
        del ws
        xkw = {"exchange": make_exchange(wsh)[0]} if points else {}
        def e2e_step():
            S.sks_sum_host(xh.numpy(), yh.numpy(), wh.numpy(), cfg.kind, scale, cfg.P, cfg.dir_seed, p0, p1,
                           cfg.matern_p, out=sh.numpy(), workspace=wsh, **xkw)
            if G > 1 and not points:   # (points: every rank holds its own targets' sums)
                sd = sh.to(dev, non_blocking=True)
                dist.all_reduce(sd)
                sh.copy_(sd)
        for _ in range(2):
            e2e_step()
        ke = max(3, min(args.steps, 10))
        evs2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ke)]
        if G > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for a, b in evs2:
            flush.zero_()
            a.record(stream)
            e2e_step()
            b.record(stream)
        torch.cuda.synchronize()
        me = sum(a.elapsed_time(b) for a, b in evs2) / ke
        te = torch.tensor([me], dtype=torch.float64, device=dev)
        if G > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        me = float(te.item())
        e2e = {"value": (full.N + full.M) * full.P / (me * 1e-3), "unit": UNIT, "ms_per_step": me,
               "h2d_bytes_per_step": 4 * (cfg.N * cfg.d + cfg.M * cfg.d + cfg.N),
               "d2h_bytes_per_step": 4 * cfg.M, "api": "sks_sum_host (pinned host buffers)",
               "bytes": "per rank"}

    if rank != 0:
        if G > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of every kernel, headline = the dominant one (live CUDA-event durations, timed region)
    pk = peaks()
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps} for k, v in prof.items()
               if v[1] > 0}
    np_local = p1 - p0
    P_launch = plan["slice_batch"] if plan.get("slice_batch", 0) else np_local
    traffic_all = {}
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")
    if os.path.exists(tpath):
        traffic_all = json.load(open(tpath))
    for k, v in kernels.items():
        if k == "aux":
            continue
        lps = max(1e-9, v["launches_per_step"])
        r = roofline(k, cfg, P_launch, plan, v["ms_per_step"] / lps, pk,
                     traffic_all[k] / lps if isinstance(traffic_all.get(k), (int, float)) else None)
        v["roofline_frac"] = r["frac"]
        v["bound"] = r["bound"]
    # headline: the dominant top-level stage; the sort path's four kernels run on two streams and overlap,
    # so the stage (fork to join on the caller's stream) is the unit, its kernels are itemised in "kernels"
    dom = max((k for k in kernels if k != "aux" and not k.startswith("sp_")), key=lambda k: kernels[k]["ms_per_step"])
    lps = max(1e-9, kernels[dom]["launches_per_step"])
    roof = roofline(dom, cfg, P_launch, plan, kernels[dom]["ms_per_step"] / lps, pk,
                    traffic_all[dom] / lps if isinstance(traffic_all.get(dom), (int, float)) else None)
    roof["share_of_step"] = kernels[dom]["ms_per_step"] / ms
    roof["ncu"] = ncu_context(cfg.name, dom)

    cpu = None
    if not args.no_cpu_baseline and G == 1:
        v, cores, desc, _ = oracle_sample(cfg, param, x, y, w, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_dict(full, param, G, points), "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": int(plan.get("launches", 0)) * args.steps, "clocks": clk,
            "mode": args.mode, "kernels_from": kernels_from, "kernels": kernels, "plan": plan}
    print(json.dumps(line), flush=True)
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
