"""Seeded synthetic inputs shared by the tests, the bench and the oracle.

This module holds NO arithmetic of the method: it only draws x, y, w (and the workload's
kernel parameter, defined by BASELINE.json as a median pairwise distance) for the five
BASELINE.json configs and the paper's own Sec. 4.1 workload.  Recipes: DESIGN.md
"Input recipe".  The paper measures only on synthetic Gaussian data; the
image-shaped cfg3/cfg4 are synthetic stand-ins with the shapes/value distributions BASELINE.json
names (no dataset is used or reproduced).

Large configs are generated in row blocks, each block from its own seeded stream, so that any
subset of rows can be regenerated without materialising the whole matrix.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

BLOCK_ROWS = 1 << 16


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    kind: str          # gaussian | negdist | laplacian | matern
    d: int
    N: int
    M: int
    P: int
    data_seed: int
    dir_seed: int
    data: str          # recipe name
    weights: str       # recipe name
    param: Optional[float] = None   # sigma / ell / beta; None -> median pairwise distance
    matern_p: int = 1
    gpus: int = 1      # GPUs the BASELINE config is quoted on


CONFIGS = {
    # BASELINE.json configs[0..4]
    "cfg1": Config("cfg1", "gaussian", 3, 1000, 1000, 64, 1, 101, "normal", "pm1", param=1.0),
    "cfg2": Config("cfg2", "negdist", 50, 100_000, 100_000, 256, 2, 102, "normal_shift05", "u01_norm"),
    "cfg3": Config("cfg3", "gaussian", 784, 60_000, 60_000, 1024, 3, 103, "grey_sparse", "inv_n"),
    "cfg4": Config("cfg4", "laplacian", 3072, 50_000, 50_000, 1024, 4, 104, "uniform01", "pm1"),
    "cfg5": Config("cfg5", "gaussian", 100, 10_000_000, 10_000_000, 512, 5, 105, "mixture10", "pm1", gpus=8),
    # the paper's Sec. 4.1 workload: N(0, 0.1^2 I), d=50, w ~ U[0,1]
    "paper_gauss": Config("paper_gauss", "gaussian", 50, 10_000, 10_000, 256, 6, 106, "normal01", "u01", param=1.0),
    "paper_matern": Config("paper_matern", "matern", 50, 10_000, 10_000, 256, 7, 107, "normal01", "u01", param=1.0,
                           matern_p=1),
    "paper_negdist": Config("paper_negdist", "negdist", 50, 10_000, 10_000, 256, 8, 108, "normal01", "u01"),
    "paper_laplace": Config("paper_laplace", "laplacian", 50, 10_000, 10_000, 256, 9, 109, "normal01", "u01",
                            param=2.0),   # alpha = 0.5 in the paper's rate convention -> ell = 2
}


def _rng(seed: int, stream: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, block])))


def _mixture_means(seed: int, d: int) -> np.ndarray:
    # 10 means ~ N(0, 4 I) = 2 * N(0, I), shared by X and Y (R12)
    return 2.0 * _rng(seed, 99, 0).standard_normal((10, d))


def _rows(recipe: str, seed: int, stream: int, d: int, r0: int, r1: int) -> np.ndarray:
    """rows [r0, r1) of a point set (stream 0 = X, 1 = Y), fp32."""
    out = np.empty((r1 - r0, d), dtype=np.float32)
    b0, b1 = r0 // BLOCK_ROWS, (r1 - 1) // BLOCK_ROWS
    for b in range(b0, b1 + 1):
        lo, hi = b * BLOCK_ROWS, (b + 1) * BLOCK_ROWS
        g = _rng(seed, stream, b)
        n = BLOCK_ROWS
        if recipe == "normal":
            blk = g.standard_normal((n, d))
        elif recipe == "normal01":
            blk = 0.1 * g.standard_normal((n, d))
        elif recipe == "normal_shift05":
            blk = g.standard_normal((n, d)) + (0.5 if stream == 1 else 0.0)
        elif recipe == "grey_sparse":
            v = g.random((n, d))
            keep = g.random((n, d)) >= 0.7
            blk = np.where(keep, v, 0.0)
        elif recipe == "uniform01":
            blk = g.random((n, d))
        elif recipe == "mixture10":
            mu = _mixture_means(seed, d)
            lab = g.integers(0, 10, size=n)
            blk = mu[lab] + g.standard_normal((n, d))
        else:
            raise ValueError(recipe)
        s0, s1 = max(lo, r0), min(hi, r1)
        out[s0 - r0:s1 - r0] = blk[s0 - lo:s1 - lo].astype(np.float32)
    return out


def points(cfg: Config, which: str, r0: int = 0, r1: Optional[int] = None) -> np.ndarray:
    n = cfg.N if which == "x" else cfg.M
    r1 = n if r1 is None else r1
    return _rows(cfg.data, cfg.data_seed, 0 if which == "x" else 1, cfg.d, r0, r1)


def rows_at(cfg: Config, which: str, idx: np.ndarray) -> np.ndarray:
    """rows idx (any order) of X or Y, generating each needed row block once."""
    idx = np.asarray(idx, dtype=np.int64)
    out = np.empty((idx.size, cfg.d), dtype=np.float32)
    blocks = idx // BLOCK_ROWS
    for b in np.unique(blocks):
        sel = np.nonzero(blocks == b)[0]
        lo = int(b) * BLOCK_ROWS
        n = cfg.N if which == "x" else cfg.M
        blk = points(cfg, which, lo, min(lo + BLOCK_ROWS, n))
        out[sel] = blk[idx[sel] - lo]
    return out


def weights(cfg: Config) -> np.ndarray:
    g = _rng(cfg.data_seed, 2, 0)
    N = cfg.N
    if cfg.weights == "pm1":
        w = g.uniform(-1.0, 1.0, N)
    elif cfg.weights == "u01":
        w = g.random(N)
    elif cfg.weights == "u01_norm":
        w = g.random(N)
        w = w / w.sum()          # normalised in fp64, then stored fp32
    elif cfg.weights == "inv_n":
        w = np.full(N, 1.0 / N)
    else:
        raise ValueError(cfg.weights)
    return w.astype(np.float32)


def median_pairwise_distance(cfg: Config, n_sub: int = 1000) -> float:
    """Workload parameter of cfg3/cfg4/cfg5 (BASELINE.json): median ||a-b|| over all pairs of a
    seeded 1000-point subsample of X u Y, fp64 (R10/R11)."""
    g = _rng(cfg.data_seed, 3, 0)
    idx = np.sort(g.choice(cfg.N + cfg.M, size=n_sub, replace=False))
    S = np.concatenate([rows_at(cfg, "x", idx[idx < cfg.N]),
                        rows_at(cfg, "y", idx[idx >= cfg.N] - cfg.N)]).astype(np.float64)
    dists = []
    for a in range(n_sub - 1):
        dd = S[a + 1:] - S[a]
        dists.append(np.sqrt(np.einsum("ij,ij->i", dd, dd)))
    return float(np.median(np.concatenate(dists)))


def kernel_param(cfg: Config) -> float:
    return float(cfg.param) if cfg.param is not None else median_pairwise_distance(cfg)


def target_subset(M: int, n: int, seed: int = 12345) -> np.ndarray:
    """seeded uniform subset of target indices (always includes 0 and M-1: ragged-tail coverage)."""
    g = _rng(seed, 4, M)
    if n >= M:
        return np.arange(M, dtype=np.int64)
    idx = g.choice(M, size=n, replace=False)
    idx[0], idx[-1] = 0, M - 1
    return np.unique(idx).astype(np.int64)


def scaled(cfg: Config, N: Optional[int] = None, M: Optional[int] = None, P: Optional[int] = None) -> Config:
    """same recipe at a smaller size (parity cases the oracle finishes in seconds)."""
    return dataclasses.replace(cfg, N=N or cfg.N, M=M or cfg.M, P=P or cfg.P)
