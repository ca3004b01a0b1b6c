"""GPU parity: the CUDA path (through the C-ABI) against the CPU fp64 oracle (-m gpu).

Metric (BASELINE.json north_star): max|s_gpu - s_oracle| / sum|w_n| against oracle (b), the sliced
estimator on the same seeded directions with direct 1D sums.  Tolerances (north_star, R15):
1e-5 for the sorting path (negdist), 1e-4 for the Fourier paths (Gaussian, Matern) and the
combined Laplacian path.  Sizes: small cases the oracle finishes in seconds spanning several tiles
and ragged tails, plus BASELINE.json's full sizes on sampled targets.
"""
import numpy as np
import pytest

import oracle as O
from paper_2401_08260_b200 import inputs as I

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_08260_b200 as S  # noqa: E402

TOL = {"negdist": 1e-5, "gaussian": 1e-4, "matern": 1e-4, "laplacian": 1e-4}
# row a1 (reading R2): max |z_gpu - z_fp64| <= 5e-7 max ||pt|| for the default variant up to
# d = 1536.  Every variant leaves a per-coordinate split residual of at most 2^-22 |x_j| (TF32x2 with the lo piece
# rounded to nearest, FP16x2) or 2^-24 |x_j| (BF16x3).  Beyond that, the tensor core's fp32 accumulator truncates at
# every MMA step (measured: a systematic shrink of |z| by ~2^-26 per step, tools/proj_error.py), so at large d the
# bound grows with the number S of accumulation steps (R2):
#     |dz| <= 2^-22 sum_j |x_j xi_j| + 2^-23 (S max_k |Z_k| + |z|),   Z_k = the partial sums after step k
PROJ_TOL = 5e-7
PROJ_TOL_MAX_D = 1536
K_STEP = {"tf32x2": (8, 2, 32), "fp16x2": (16, 2, 64), "bf16x3": (16, 3, 64)}   # (K per MMA, pieces, k-block)


def default_projection(d, aligned=True):
    return ("fp16x2" if d >= 256 else "tf32x2") if (aligned and d % 4 == 0) else ("tf32x2" if d < 256 else "bf16x3")


def proj_bound(pts, xi, mode):
    """the per-(slice, point) bound above; pts (n, d), xi (P, d) fp64 -> (P, n)"""
    kstep, pieces, kblk = K_STEP[mode]
    d = pts.shape[1]
    dp = -(-d // kblk) * kblk
    steps = pieces * dp // kstep
    x = pts.astype(np.float64)
    prods = xi[:, None, :] * x[None, :, :]                       # (P, n, d)
    pad = np.zeros(prods.shape[:2] + (dp - d,))
    part = np.cumsum(np.concatenate([prods, pad], 2).reshape(prods.shape[:2] + (dp // kstep, kstep)).sum(3), 2)
    zmax = np.abs(part).max(2)
    return 2.0**-22 * np.abs(prods).sum(2) + 2.0**-23 * (steps * zmax + np.abs(part[:, :, -1]))


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2401_08260_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(got, ref, w):
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / np.abs(w.astype(np.float64)).sum())


# ---------------------------------------------------------------- a1: projection
@pytest.mark.parametrize("n,d,P", [(1, 3, 1), (300, 3, 64), (1000, 50, 70), (257, 784, 33), (129, 3072, 17),
                                   # > 128 slices at d >= 256: FP16x2 on CTA pairs (k_proj_pair), ragged slice and
                                   # point tiles, a pair tile whose second CTA holds no points
                                   (3001, 784, 300), (1000, 3072, 257), (300, 256, 512)])
def test_projection_parity(n, d, P):
    rng = np.random.default_rng(n + d)
    pts = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    z = S.sks_project(dev(pts), P, seed=7).cpu().numpy()
    zo = O.project(pts, O.unit_directions(P, d, 7))
    scale = np.linalg.norm(pts.astype(np.float64), axis=1).max()
    if d <= PROJ_TOL_MAX_D:
        assert np.max(np.abs(z - zo)) <= PROJ_TOL * scale, np.max(np.abs(z - zo)) / scale
    bound = proj_bound(pts, O.unit_directions(P, d, 7), default_projection(d))
    assert np.all(np.abs(z - zo) <= bound), np.max(np.abs(z - zo) / bound)


# ---------------------------------------------------------------- a2-a7: the 1D engines on given projections
CASES_1D = [
    # kind, scale, d, N, M, S
    ("negdist", 0.0, 50, 3001, 1537, 5),
    ("negdist", 0.0, 3, 1, 1, 2),
    ("negdist", 0.0, 3, 70000, 333, 2),
    ("negdist", 0.0, 50, 200000, 400, 2),   # ~58 owners per slice (sortpart.cu)
    ("negdist", 0.0, 50, 600000, 200, 2),   # > 128 owners: plan bases, atomic-free partition, global owner table
    ("negdist", 0.0, 50, 5000000, 300, 1),  # > 1024 owners (1437): the many-owner partition with 1024-thread CTAs
    ("gaussian", 1.0, 3, 2003, 1001, 4),
    ("gaussian", 11.0, 784, 4097, 515, 3),
    ("gaussian", 30.0, 100, 5000, 700, 3),
    ("laplacian", 22.6, 3072, 3001, 517, 3),
    ("laplacian", 2.0, 50, 2500, 600, 3),
    ("matern", 8.0, 50, 3000, 600, 3),    # beta large enough that the oracle's 1F2 series stays well
    ("matern", 5.0, 10, 2000, 300, 2),    # conditioned over the test's |dz| range
    ("matern", 1.0, 3, 1500, 400, 2),     # d = 3: the oracle's closed form (Cor 2.4), any beta (the paper's beta = 1)
    ("laplacian", 0.5, 3, 2000, 500, 2),  # d = 3 closed form (Cor 2.4) far beyond the series' range (|dz| / ell ~ 12)
    ("gaussian", 0.3, 3, 2000, 500, 2),
]


@pytest.mark.parametrize("kind,scale,d,N,M,nsl", CASES_1D)
def test_sum_1d_parity(kind, scale, d, N, M, nsl):
    rng = np.random.default_rng(N + M + d)
    spread = {3: 1.0, 10: 1.0, 50: 1.0, 100: 2.2, 784: 0.28, 3072: 0.29}[d]
    zx = (spread * rng.standard_normal((nsl, N))).astype(np.float32)
    zy = (spread * rng.standard_normal((nsl, M)) + 0.1).astype(np.float32)
    w = rng.uniform(-1, 1, N).astype(np.float32)
    t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), d, kind, scale if scale else 1.0).cpu().numpy()
    for q in range(nsl):
        ref = O.sum_1d(kind, scale, d, zx[q].astype(np.float64), w.astype(np.float64), zy[q].astype(np.float64))
        err = rel_err(t[q], ref, w)
        assert err <= TOL[kind], (q, err)


@pytest.mark.parametrize("engine", ["nfft", "ndft"])
@pytest.mark.parametrize("kind,scale,d,N,M,nsl", [c for c in CASES_1D if c[0] in ("gaussian", "matern")])
def test_sum_1d_engines(kind, scale, d, N, M, nsl, engine):
    # both Fourier engines (NFFT: Remark P:519-525; NDFT on the kept band: P:508-517) against oracle (b)
    rng = np.random.default_rng(N + M + d + 1)
    spread = {3: 1.0, 10: 1.0, 50: 1.0, 100: 2.2, 784: 0.28, 3072: 0.29}[d]
    zx = (spread * rng.standard_normal((nsl, N))).astype(np.float32)
    zy = (spread * rng.standard_normal((nsl, M)) - 0.05).astype(np.float32)
    w = rng.uniform(-1, 1, N).astype(np.float32)
    try:
        t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), d, kind, scale, engine=engine).cpu().numpy()
    except S.SKSError as e:   # NDFT refuses bands wider than 32 coefficients
        assert engine == "ndft" and e.status == 2, e
        pytest.skip(f"band too wide for the NDFT: {e}")
    info = S.sks_last_plan()
    assert info["engine"] == (2 if engine == "ndft" else 1)
    for q in range(nsl):
        ref = O.sum_1d(kind, scale, d, zx[q].astype(np.float64), w.astype(np.float64), zy[q].astype(np.float64))
        assert rel_err(t[q], ref, w) <= TOL[kind], (q, engine, rel_err(t[q], ref, w))


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg5", "paper_gauss", "paper_matern"])
def test_ndft_engine_end_to_end(name):
    # Alg. 1 with the NDFT engine on the BASELINE-shaped Gaussian workloads, against oracle (b)
    size = {"cfg1": {}, "cfg3": dict(N=3000, M=600, P=8), "cfg5": dict(N=20000, M=1000, P=8),
            "paper_gauss": dict(N=3000, M=600, P=16), "paper_matern": dict(N=3000, M=600, P=16)}[name]
    cfg = I.scaled(I.CONFIGS[name], **size) if size else I.CONFIGS[name]
    try:
        _, got, ref, w, _ = run_cfg(cfg, n_tgt=200, engine="ndft")
    except S.SKSError as e:
        assert e.status == 2, e
        pytest.skip(f"band too wide for the NDFT: {e}")
    info = S.sks_last_plan()
    assert info["engine"] == 2 and info["band_width"] <= 32, info
    assert rel_err(got, ref, w) <= TOL[cfg.kind], rel_err(got, ref, w)
    run_cfg(cfg, n_tgt=10)
    assert S.sks_last_plan()["engine"] == 1   # auto = NFFT


def test_sum_1d_degenerate_identical_points():
    # all sources at one point (zero range) and targets on top of it / away from it
    N, M = 1000, 300
    zx = np.full((2, N), 0.75, np.float32)
    zy = np.concatenate([np.full((2, 100), 0.75), np.linspace(-2, 3, 200)[None].repeat(2, 0)], 1).astype(np.float32)
    w = np.random.default_rng(0).random(N).astype(np.float32)
    for kind, scale, d in [("negdist", 1.0, 5), ("gaussian", 1.0, 5), ("laplacian", 1.0, 5)]:
        t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), d, kind, scale).cpu().numpy()
        for q in range(2):
            ref = O.sum_1d(kind, scale if kind != "negdist" else 0.0, d, zx[q].astype(np.float64),
                           w.astype(np.float64), zy[q].astype(np.float64))
            assert rel_err(t[q], ref, w) <= TOL[kind], kind


def test_sum_1d_owner_overflow_multipass():
    # more identical sources than one owner's shared memory holds (8192): that owner runs several passes over
    # subsets of its sources (sortpart.cu S3); the rest of the slice is spread normally
    rng = np.random.default_rng(11)
    N, M = 21000, 600
    zx = np.stack([np.concatenate([np.full(13000, 0.3), rng.standard_normal(8000)]),
                   np.concatenate([rng.standard_normal(8000), np.full(13000, -1.25)])]).astype(np.float32)
    zy = np.stack([np.concatenate([np.full(50, 0.3), rng.standard_normal(550)]),
                   np.concatenate([np.full(50, -1.25), rng.standard_normal(550)])]).astype(np.float32)
    w = rng.uniform(-1, 1, N).astype(np.float32)
    for kind, scale in [("negdist", 1.0), ("laplacian", 2.0)]:
        t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), 50, kind, scale).cpu().numpy()
        for q in range(2):
            ref = O.sum_1d(kind, scale if kind != "negdist" else 0.0, 50, zx[q].astype(np.float64),
                           w.astype(np.float64), zy[q].astype(np.float64))
            assert rel_err(t[q], ref, w) <= TOL[kind], (kind, q)


@pytest.mark.slow
def test_sum_1d_sequential_plan_bases():
    # k_sp_hist's one-chunk-at-a-time plan bases (base_par = 0): > 128 owners and 2 (NH + 1) + G + 1 + chunks * G
    # beyond the shared-memory plan budget.  N = 4e6 (G = 1150 owners, NH = 16384) with M = 262144 targets (8 + 8
    # histogram chunks): 32770 + 1151 + 16 * 1150 = 52321 > 51200 ints.  Checked on a target subset
    rng = np.random.default_rng(13)
    N, M = 4_000_000, 262_144
    zx = rng.standard_normal((1, N)).astype(np.float32)
    zy = (1.3 * rng.standard_normal((1, M))).astype(np.float32)
    w = rng.uniform(0, 1, N).astype(np.float32)
    t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), 50, "negdist", 1.0).cpu().numpy()
    sub = np.linspace(0, M - 1, 300).astype(np.int64)
    ref = O.sum_1d("negdist", 0.0, 50, zx[0].astype(np.float64), w.astype(np.float64), zy[0, sub].astype(np.float64))
    assert rel_err(t[0, sub], ref, w) <= TOL["negdist"]


def test_sum_1d_targets_outside_source_range():
    # targets below / above every source (clamped to the first / last owner and bucket); |t| stays within
    # ~100 sum|w| so that the fp32 output itself resolves 1e-5 sum|w|
    rng = np.random.default_rng(12)
    N, M = 9000, 400
    zx = rng.standard_normal((2, N)).astype(np.float32)
    zy = np.concatenate([rng.uniform(-10, -5, (2, 200)), rng.uniform(5, 10, (2, 200))], 1).astype(np.float32)
    w = rng.uniform(0, 1, N).astype(np.float32)
    t = S.sks_sum_1d(dev(zx), dev(zy), dev(w), 50, "negdist", 1.0).cpu().numpy()
    for q in range(2):
        ref = O.sum_1d("negdist", 0.0, 50, zx[q].astype(np.float64), w.astype(np.float64), zy[q].astype(np.float64))
        assert rel_err(t[q], ref, w) <= TOL["negdist"]


# ---------------------------------------------------------------- end to end (Alg. 1) vs oracle (b)
def run_cfg(cfg, n_tgt=None, p0=0, p1=None, **opts):
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    param = I.kernel_param(cfg)
    s = S.sks_sum(dev(x), dev(y), dev(w), cfg.kind, param if cfg.kind != "negdist" else 1.0, cfg.P, cfg.dir_seed,
                  p_begin=p0, p_end=p1, matern_p=cfg.matern_p, **opts).cpu().numpy()
    tgt = I.target_subset(cfg.M, n_tgt) if n_tgt else np.arange(cfg.M)
    ref = O.sliced_sum(cfg.kind, param if cfg.kind != "negdist" else 0.0, x, y, w, cfg.P, cfg.dir_seed, targets=tgt,
                       p0=p0, p1=p1, matern_p=cfg.matern_p)
    return s, s[tgt], ref, w, (x, y, param, tgt)


SMALL = [
    ("cfg1", {}),                                               # full BASELINE configs[0]
    ("cfg2", dict(N=20000, M=4000, P=24)),
    ("cfg3", dict(N=6000, M=1200, P=16)),
    ("cfg4", dict(N=4000, M=800, P=8)),
    ("cfg5", dict(N=30000, M=2000, P=16)),
    ("paper_gauss", dict(N=3000, M=1000, P=32)),
    ("paper_matern", dict(N=3000, M=1000, P=32)),
    ("paper_negdist", dict(N=3000, M=1000, P=32)),
    ("paper_laplace", dict(N=3000, M=1000, P=32)),
]


@pytest.mark.parametrize("name,size", SMALL, ids=[s[0] for s in SMALL])
def test_end_to_end_small(name, size):
    cfg = I.scaled(I.CONFIGS[name], **size) if size else I.CONFIGS[name]
    _, got, ref, w, _ = run_cfg(cfg, n_tgt=min(cfg.M, 400))
    err = rel_err(got, ref, w)
    print(f"{name}: max|ds|/sum|w| = {err:.3e}  plan={S.sks_last_plan()}")
    assert err <= TOL[cfg.kind], err


def test_slice_ranges_add_up():
    # the multi-GPU contract: partial ranges sum (one all-reduce) to the full estimate (north_star)
    cfg = I.scaled(I.CONFIGS["cfg2"], N=5000, M=1000, P=32)
    full = run_cfg(cfg, n_tgt=50)[0]
    a = run_cfg(cfg, n_tgt=50, p0=0, p1=12)[0]
    b = run_cfg(cfg, n_tgt=50, p0=12, p1=32)[0]
    w = I.weights(cfg)
    assert rel_err(a + b, full.astype(np.float64), w) <= 1e-6
    cfg = I.scaled(I.CONFIGS["cfg3"], N=3000, M=500, P=8)
    full = run_cfg(cfg, n_tgt=50)[0]
    parts = sum(run_cfg(cfg, n_tgt=50, p0=q, p1=q + 2)[0].astype(np.float64) for q in range(0, 8, 2))
    assert rel_err(parts, full.astype(np.float64), I.weights(cfg)) <= 1e-6


def test_slice_batching_invariance():
    cfg = I.scaled(I.CONFIGS["paper_laplace"], N=2000, M=500, P=20)
    a = run_cfg(cfg, n_tgt=20)[0]
    b = run_cfg(cfg, n_tgt=20, slice_batch=7)[0]
    assert rel_err(a, b.astype(np.float64), I.weights(cfg)) <= 1e-6


def test_host_entry_point_matches_device():
    cfg = I.scaled(I.CONFIGS["cfg2"], N=3000, M=700, P=16)
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    s_dev = S.sks_sum(dev(x), dev(y), dev(w), "negdist", 1.0, cfg.P, cfg.dir_seed).cpu().numpy()
    s_host = S.sks_sum_host(x, y, w, "negdist", 1.0, cfg.P, cfg.dir_seed)
    assert rel_err(s_host, s_dev.astype(np.float64), w) <= 1e-6


def test_errors_fail_loudly():
    x = torch.randn(100, 4, device="cuda")
    y = torch.randn(30, 4, device="cuda")
    w = torch.rand(100, device="cuda")
    x[5, 1] = float("nan")
    for kind in ("negdist", "gaussian"):
        with pytest.raises(S.SKSError) as e:
            S.sks_sum(x, y, w, kind, 1.0, 8, 1)
        assert e.value.status == 5
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(S.SKSError) as e:
        S.sks_sum(torch.randn(100, 4, device="cuda"), y, w, "negdist", 1.0, 8, 1, workspace=ws)
    assert e.value.status == 4
    # d >= 256 (FP16x2): an Inf / NaN input trips the trap, the call reruns on TF32x2, which reports it
    xb = torch.randn(300, 256, device="cuda")
    yb = torch.randn(40, 256, device="cuda")
    wb = torch.rand(300, device="cuda")
    for bad in (float("inf"), float("nan")):
        xb2 = xb.clone()
        xb2[7, 3] = bad
        for kind in ("negdist", "gaussian"):
            with pytest.raises(S.SKSError) as e:
                S.sks_sum(xb2, yb, wb, kind, 20.0, 8, 1)
            assert e.value.status == 5, (bad, kind)


# ---------------------------------------------------------------- BASELINE.json full sizes, sampled targets
FULL = [("cfg2", 256), ("cfg3", 256), ("cfg4", 256)]


@pytest.mark.slow
@pytest.mark.parametrize("name,n_tgt", FULL, ids=[f[0] for f in FULL])
def test_full_size_sampled(name, n_tgt):
    cfg = I.CONFIGS[name]
    _, got, ref, w, _ = run_cfg(cfg, n_tgt=n_tgt)
    err = rel_err(got, ref, w)
    print(f"{name} FULL: max|ds|/sum|w| = {err:.3e}  plan={S.sks_last_plan()}")
    assert err <= TOL[cfg.kind], err


@pytest.mark.slow
def test_cfg5_slice_subset_sampled():
    # cfg5 at full N = M = 1e7 on one GPU: a 2-slice sub-range at the start of each of the 8 ranks' ranges (16 slices
    # spanning all 8 rank ranges, in the launch configuration of a rank: p_begin/p_end), 32 sampled targets each
    from paper_2401_08260_b200.parallel import slice_range
    cfg = I.CONFIGS["cfg5"]
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    param = I.kernel_param(cfg)
    xd, yd, wd = dev(x), dev(y), dev(w)
    tgt = I.target_subset(cfg.M, 32)
    for rank in range(8):
        p0 = slice_range(rank, 8, cfg.P)[0]
        s = S.sks_sum(xd, yd, wd, "gaussian", param, cfg.P, cfg.dir_seed, p_begin=p0, p_end=p0 + 2).cpu().numpy()
        ref = O.sliced_sum("gaussian", param, x, y, w, cfg.P, cfg.dir_seed, targets=tgt, p0=p0, p1=p0 + 2)
        # the 2-slice partial is (1/P) * sum of 2 slices: compare on the per-slice-mean scale
        err = rel_err(s[tgt] * cfg.P / 2, ref * cfg.P / 2, w)
        print(f"cfg5 rank {rank} slices [{p0}, {p0 + 2}): max|ds|/sum|w| = {err:.3e}")
        assert err <= TOL["gaussian"], (rank, err)


# ---------------------------------------------------------------- the paper's error claims on the GPU path
def test_slicing_error_decays_like_inverse_sqrt_P():
    # Prop. 2.6 / Thm 2.7: the per-summand error of the GPU estimate against the exact sum
    # (oracle (a)) decays like P^{-1/2}; the paper's Sec. 4.1 workload, Gaussian sigma = 1
    cfg = I.scaled(I.CONFIGS["paper_gauss"], N=3000, M=3000)
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    tgt = I.target_subset(cfg.M, 200)
    exact = O.exact_sum("gaussian", 1.0, x, y[tgt], w)
    sw = np.abs(w.astype(np.float64)).sum()
    Ps = [16, 64, 256, 1024]
    errs = []
    for P in Ps:
        s = S.sks_sum(dev(x), dev(y), dev(w), "gaussian", 1.0, P, cfg.dir_seed).cpu().numpy()
        errs.append(np.abs(s[tgt] - exact).sum() / (len(tgt) * sw))
    slope = np.polyfit(np.log(Ps), np.log(errs), 1)[0]
    assert -0.75 < slope < -0.3, (slope, errs)


def test_many_slices_projection_chunks():
    # more slices than one projection launch takes (1024): chunked launches, same result as slice ranges
    cfg = I.scaled(I.CONFIGS["paper_gauss"], N=600, M=300, P=2500)
    s_all = run_cfg(cfg, n_tgt=50)[0].astype(np.float64)
    s_a = run_cfg(cfg, n_tgt=50, p0=0, p1=1300)[0].astype(np.float64)
    s_b = run_cfg(cfg, n_tgt=50, p0=1300, p1=2500)[0].astype(np.float64)
    assert rel_err(s_a + s_b, s_all, I.weights(cfg)) <= 1e-6


@pytest.mark.parametrize("mode", ["bf16x3", "tf32x2", "fp16x2"])
def test_projection_modes(mode):
    # every row-a1 variant (R2) against the fp64 projection, at small and large d (sks_options.projection)
    for n, d, P in [(300, 3, 64), (1000, 50, 70), (257, 784, 33), (129, 3072, 17), (700, 100, 300), (333, 52, 9),
                    (100, 258, 5)]:
        pts = np.random.default_rng(n + d).uniform(-1, 1, (n, d)).astype(np.float32)
        z = S.sks_project(dev(pts), P, seed=7, projection=mode).cpu().numpy()
        zo = O.project(pts, O.unit_directions(P, d, 7))
        scale = np.linalg.norm(pts.astype(np.float64), axis=1).max()
        err = np.max(np.abs(z - zo)) / scale
        eff = mode if (mode != "fp16x2" or d % 4 == 0) else "tf32x2"   # FP16x2 needs TMA-readable points
        assert np.all(np.abs(z - zo) <= proj_bound(pts, O.unit_directions(P, d, 7), eff)), (mode, n, d, P, err)
        if d <= 100:
            assert err <= PROJ_TOL, (mode, n, d, P, err)
    # the end-to-end sum on a forced variant
    cfg = I.scaled(I.CONFIGS["cfg2"], N=3000, M=500, P=8)
    _, got, ref, w, _ = run_cfg(cfg, n_tgt=100, projection=mode)
    assert rel_err(got, ref, w) <= TOL["negdist"]


def test_fp16x2_default_scaling_and_range_fallback():
    # d >= 256 runs FP16x2 (proj_mode 4): points scaled by a power of two from a row sample; data far from 1 in
    # magnitude must keep fp32-accurate projections (the sums match oracle (b) exactly for negdist), and a row
    # outside the sampled range (beyond the fp16 range; row 1 is not among the sampled rows k L / 1024) makes the call
    # rerun on TF32x2 (proj_mode 3) with the same result
    rng = np.random.default_rng(5)
    N, M, d, P = 5000, 400, 256, 6
    base_x = rng.normal(size=(N, d)).astype(np.float32)
    base_y = rng.normal(size=(M, d)).astype(np.float32)
    w = rng.uniform(0, 1, N).astype(np.float32)
    tgt = np.arange(0, M, 7)
    for mag, spike, mode in [(1e-5, False, 4), (1.0, False, 4), (3e4, False, 4), (1.0, True, 3)]:
        x = base_x * np.float32(mag)
        y = base_y * np.float32(mag)
        if spike:
            x[1] *= np.float32(1e5)
        s = S.sks_sum(dev(x), dev(y), dev(w), "negdist", 1.0, P, 11).cpu().numpy()
        assert S.sks_last_plan()["proj_mode"] == mode, (mag, spike, S.sks_last_plan())
        ref = O.sliced_sum("negdist", 0.0, x, y, w, P, 11, targets=tgt)
        # negdist is homogeneous of degree 1: compare relative to mag (and to the spike's scale)
        err = np.max(np.abs(s[tgt].astype(np.float64) - ref)) / np.abs(ref).max()
        assert err <= 2e-6, (mag, spike, err)


@pytest.mark.parametrize("N,M,d,kind", [(100, 50, 784, "negdist"), (130, 7, 256, "gaussian"), (3, 2, 300, "negdist"),
                                        (1000, 500, 258, "negdist"), (129, 129, 512, "laplacian")])
def test_projection_paths_small_shapes(N, M, d, kind):
    # the projection variants at awkward sizes: a single straddling point tile (N < 128), d = 256 (FP16x2 from
    # d >= 256), d % 4 != 0 above 256 (BF16x3 with the split pass), tiny N / M
    rng = np.random.default_rng(N * 7 + d)
    x = rng.normal(size=(N, d)).astype(np.float32)
    y = rng.normal(size=(M, d)).astype(np.float32)
    w = rng.uniform(-1, 1, N).astype(np.float32)
    P, scale = 8, 25.0
    s = S.sks_sum(dev(x), dev(y), dev(w), kind, scale, P, 3).cpu().numpy()
    ref = O.sliced_sum(kind, scale if kind != "negdist" else 0.0, x, y, w, P, 3)
    err = rel_err(s, ref, w)
    tol = TOL[kind]
    if kind == "negdist":
        # exact up to the projections' rounding (R2: |dz| <= PROJ_TOL ||pt||): |dt| <= c_d sum|w| 2 PROJ_TOL max||pt||
        import math
        cd = math.sqrt(math.pi) * math.exp(math.lgamma((d + 1) / 2) - math.lgamma(d / 2))
        tol = max(tol, 2 * PROJ_TOL * cd * max(np.linalg.norm(x, axis=1).max(), np.linalg.norm(y, axis=1).max()))
    assert err <= tol, (N, M, d, kind, err, tol, S.sks_last_plan())


# ---------------------------------------------------------------- asynchronous calls and CUDA-graph replay
@pytest.mark.parametrize("name,size", [("cfg1", {}), ("cfg2", dict(N=20000, M=3000, P=16)),
                                       ("paper_laplace", dict(N=3000, M=800, P=16)),
                                       ("cfg3", dict(N=3000, M=600, P=16))], ids=["cfg1", "cfg2", "laplace", "cfg3"])
def test_async_and_graph_calls(name, size):
    # the whole call is enqueued without a host synchronisation (device planner, predicated rerun); async calls and
    # graph replays give the synchronous call's result, and a replay picks up new input values in the same buffers
    cfg = I.scaled(I.CONFIGS[name], **size) if size else I.CONFIGS[name]
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    param = I.kernel_param(cfg) if cfg.kind != "negdist" else 1.0
    xd, yd, wd = dev(x), dev(y), dev(w)
    ws = torch.empty(S.sks_workspace_size(cfg.N, cfg.M, cfg.d, cfg.kind, param, cfg.P), dtype=torch.uint8,
                     device="cuda")
    args = (cfg.kind, param, cfg.P, cfg.dir_seed)
    ref = S.sks_sum(xd, yd, wd, *args, workspace=ws).cpu().numpy().astype(np.float64)
    a = S.sks_sum(xd, yd, wd, *args, workspace=ws, async_=True)
    S.sks_sync_status(ws)
    assert rel_err(a.cpu().numpy(), ref, w) <= 1e-6
    out = torch.empty(cfg.M, dtype=torch.float32, device="cuda")
    for _ in range(3):   # first call: eager + capture; then replays
        S.sks_sum(xd, yd, wd, *args, out=out, workspace=ws, graph=True)
        S.sks_sync_status(ws)
        assert rel_err(out.cpu().numpy(), ref, w) <= 1e-6
    w2 = (w * np.float32(0.5)).astype(np.float32)
    wd.copy_(torch.from_numpy(w2))
    S.sks_sum(xd, yd, wd, *args, out=out, workspace=ws, graph=True)
    S.sks_sync_status(ws)
    assert rel_err(out.cpu().numpy(), 0.5 * ref, w) <= 1e-6


def test_async_status_reports_errors():
    x = torch.randn(300, 8, device="cuda")
    y = torch.randn(40, 8, device="cuda")
    w = torch.rand(300, device="cuda")
    x[3, 2] = float("nan")
    ws = torch.empty(S.sks_workspace_size(300, 40, 8, "gaussian", 1.0, 8), dtype=torch.uint8, device="cuda")
    S.sks_sum(x, y, w, "gaussian", 1.0, 8, 1, workspace=ws, async_=True)   # enqueued: no error yet
    with pytest.raises(S.SKSError) as e:
        S.sks_sync_status(ws)
    assert e.value.status == 5
    # a Gaussian far narrower than the data's range needs a grid beyond the built limit: reported, not wrong
    x = 100.0 * torch.randn(300, 8, device="cuda")
    with pytest.raises(S.SKSError) as e:
        S.sks_sum(x, y, w, "gaussian", 1e-3, 8, 1)
    assert e.value.status == 2


# ---------------------------------------------------------------- rows a1 + a5 fused (large N, Fourier kernels)
@pytest.mark.parametrize("kind,scale,d,N,M,P", [("gaussian", 30.0, 100, 300_001, 3000, 150),
                                                ("matern", 20.0, 52, 262_144 + 77, 1500, 33),
                                                ("gaussian", 2.0, 8, 400_000, 2000, 20)])
def test_fused_projection_spread(kind, scale, d, N, M, P):
    # N >= 2^18, d <= 128, d % 4 == 0: the sources' projections are spread from the tensor-core accumulators
    # (fused.cu, plan_info.fused = 1); ragged slice tiles (P % 128 != 0) and point tiles (N % 128 != 0)
    cfg = I.Config("fused", kind, d, N, M, P, 31, 131, "mixture10", "pm1", param=scale)
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    s = S.sks_sum(dev(x), dev(y), dev(w), kind, scale, P, cfg.dir_seed).cpu().numpy()
    info = S.sks_last_plan()
    assert info["fused"] == 1, info
    tgt = I.target_subset(M, 48)
    ref = O.sliced_sum(kind, scale, x, y, w, P, cfg.dir_seed, targets=tgt)
    err = rel_err(s[tgt], ref, w)
    print(f"fused {kind} d={d} N={N} P={P}: max|ds|/sum|w| = {err:.3e}  plan={info}")
    assert err <= TOL[kind], err


_WINDOW_CASE = {}


@pytest.mark.gpu
@pytest.mark.parametrize("w,os_,tol", [(5, 2, 1e-6), (5, 4, 1e-6), (4, 4, 1e-5), (7, 2, 1e-6), (10, 2, 1e-6),
                                        (6, 4, 1e-6), (4, 2, 1e-5), (6, 8, 1e-6), (5, 8, 1e-6)])
def test_fused_window_variants(w, os_, tol):
    # the fused spread's window variants: odd widths (a middle tap beside the mirror pairs), footprints beyond 32
    # cells (w = 7, 10 and oversampling 4: the kernel variant with 4 private copies of 64 cells instead of 8 of 32
    # takes the tile; oversampling 8: ~105 cells, the variant with one shared column and shared-memory atomics),
    # more than 4 mirror pairs (coefficients staged by 2 warps).  Bounds: 10x the measured errors
    cfg = I.Config("fused", "gaussian", 100, 300_001, 2000, 40, 35, 135, "mixture10", "pm1", param=30.0)
    if "case" not in _WINDOW_CASE:   # (one oracle run serves all variants)
        x, y, wt = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
        tgt = I.target_subset(cfg.M, 32)
        _WINDOW_CASE["case"] = (x, y, wt, tgt, O.sliced_sum("gaussian", 30.0, x, y, wt, cfg.P, cfg.dir_seed,
                                                            targets=tgt))
    x, y, wt, tgt, ref = _WINDOW_CASE["case"]
    s = S.sks_sum(dev(x), dev(y), dev(wt), "gaussian", 30.0, cfg.P, cfg.dir_seed, window_w=w,
                  oversample=os_).cpu().numpy()
    info = S.sks_last_plan()
    assert info["fused"] == 1 and info["window_w"] == w, info
    err = rel_err(s[tgt], ref, wt)
    print(f"fused window w={w} os={os_}: max|ds|/sum|w| = {err:.3e}  plan={info}")
    assert err <= tol, err


@pytest.mark.gpu
def test_fused_mixed_row_magnitudes():
    # the fused kernels' FP16x2 operands carry one power-of-two scale per 8-row group (fused.cu k_prep_f16): rows
    # whose magnitudes differ by up to 2^8 inside a group keep the projection's fp32 accuracy (reading R2)
    cfg = I.Config("fused", "gaussian", 100, 300_001, 3000, 40, 33, 133, "mixture10", "pm1", param=200.0)
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    rng = np.random.default_rng(7)
    x = (x * np.exp2(rng.uniform(-4, 4, size=(cfg.N, 1)))).astype(np.float32)
    y = (y * np.exp2(rng.uniform(-4, 4, size=(cfg.M, 1)))).astype(np.float32)
    s = S.sks_sum(dev(x), dev(y), dev(w), "gaussian", 200.0, cfg.P, cfg.dir_seed).cpu().numpy()
    assert S.sks_last_plan()["fused"] == 1
    tgt = I.target_subset(cfg.M, 48)
    ref = O.sliced_sum("gaussian", 200.0, x, y, w, cfg.P, cfg.dir_seed, targets=tgt)
    err = rel_err(s[tgt], ref, w)
    print(f"fused, mixed row magnitudes: max|ds|/sum|w| = {err:.3e}")
    assert err <= TOL["gaussian"], err


# ---------------------------------------------------------------- opt-in bitwise determinism
@pytest.mark.parametrize("name,size,kw", [("cfg1", {}, {}), ("cfg1", {}, {"engine": "ndft"}),
                                          ("cfg2", dict(N=30000, M=5000, P=24), {}),
                                          ("paper_laplace", dict(N=4000, M=1000, P=40), {}),
                                          ("paper_matern", dict(N=3000, M=800, P=16), {}),
                                          ("cfg5", dict(N=300_000, M=3000, P=20), {})],
                         ids=["cfg1", "cfg1-ndft", "cfg2", "laplace", "matern", "cfg5-large-N"])
def test_deterministic_mode_bitwise(name, size, kw):
    # sks_options.deterministic: no floating-point atomics, fixed-order reductions -> identical bits run to run,
    # the same estimate as the default mode (which adds per-group sums with fp64 atomics), and oracle parity
    cfg = I.scaled(I.CONFIGS[name], **size) if size else I.CONFIGS[name]
    x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
    par = I.kernel_param(cfg) if cfg.kind != "negdist" else 1.0
    xd, yd, wd = dev(x), dev(y), dev(w)
    runs = [S.sks_sum(xd, yd, wd, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, deterministic=True,
                      **kw).cpu().numpy() for _ in range(3)]
    assert all(np.array_equal(runs[0].view(np.uint32), r.view(np.uint32)) for r in runs[1:])
    assert S.sks_last_plan()["fused"] == 0
    base = S.sks_sum(xd, yd, wd, cfg.kind, par, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p, **kw).cpu().numpy()
    assert rel_err(runs[0], base.astype(np.float64), w) <= 1e-6
    tgt = I.target_subset(cfg.M, 100)
    ref = O.sliced_sum(cfg.kind, par if cfg.kind != "negdist" else 0.0, x, y, w, cfg.P, cfg.dir_seed, targets=tgt,
                       matern_p=cfg.matern_p)
    assert rel_err(runs[0][tgt], ref, w) <= TOL[cfg.kind]


def test_release_caches_then_rebuild():
    # sks_release_caches frees the cached directions, planner tables and CUDA graphs; the next calls rebuild them
    # and return the same sums (eager and graph-replayed calls)
    cfg = I.CONFIGS["cfg1"]
    x, y, w = (dev(v) for v in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
    s1 = S.sks_sum(x, y, w, "gaussian", 1.0, cfg.P, cfg.dir_seed).cpu()
    g1 = S.sks_sum(x, y, w, "gaussian", 1.0, cfg.P, cfg.dir_seed, graph=True).cpu()
    S.sks_release_caches()
    s2 = S.sks_sum(x, y, w, "gaussian", 1.0, cfg.P, cfg.dir_seed).cpu()
    g2 = S.sks_sum(x, y, w, "gaussian", 1.0, cfg.P, cfg.dir_seed, graph=True).cpu()
    S.sks_release_caches()
    assert torch.equal(s1, s2) and torch.equal(g1, g2)
    assert float((s1 - g1).abs().max()) <= 1e-6 * float(w.abs().sum())
