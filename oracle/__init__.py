"""CPU fp64 oracle for sliced fast kernel summation (arXiv 2401.08260).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2401_08260_b200``) never imports it and shares no code with it.

Thin ctypes wrapper around ``oracle/oracle.c`` (plain C, fp64, OpenMP over targets).
Every function cites the PAPER.md passage it follows; see the header of oracle.c.
Parity status: every function below is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` (no function is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KIND = {"gaussian": 0, "negdist": 1, "laplacian": 2, "matern": 3}


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -O2, OpenMP, IEEE fp64: no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i, i64, u64, vp = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        sig = {
            "or_cd": (d, [i]),
            "or_hyp1f1": (d, [d, d, d]),
            "or_hyp1f2": (d, [d, d, d, d]),
            "or_F": (d, [i, d, i, d]),
            "or_f": (d, [i, d, i, i, d]),
            "or_f_vec": (None, [i, d, i, i, vp, vp, i64]),
            "or_f_series_vec": (None, [i, d, i, i, vp, vp, i64]),
            "or_F_vec": (None, [i, d, i, vp, vp, i64]),
            "or_splitmix64": (u64, [u64]),
            "or_round_bf16": (d, [d]),
            "or_directions": (None, [i, i, u64, i, i, vp, vp]),
            "or_project": (None, [vp, i64, i, vp, i, vp]),
            "or_exact_sum": (None, [i, d, i, i, vp, i64, vp, vp, i64, vp, vp]),
            "or_sliced_sum": (None, [i, d, i, i, vp, i64, vp, vp, i64, vp, i, i, i, vp, vp]),
            "or_sum_1d": (None, [i, d, i, i, vp, vp, i64, vp, i64, vp]),
            "or_error": (i, []),
            "or_clear_error": (None, []),
            "or_num_threads": (i, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleConditioningError(RuntimeError):
    """A plain fp64 series lost too many digits to be trusted as an oracle value."""


def _check():
    if lib().or_error():
        lib().or_clear_error()
        raise OracleConditioningError("oracle series evaluation ill-conditioned (see oracle.c OR_MAX_ABS_CANCEL)")


def num_threads() -> int:
    return int(lib().or_num_threads())


def cd(d: int) -> float:
    """c_d = sqrt(pi) Gamma((d+1)/2)/Gamma(d/2), Table 1."""
    return float(lib().or_cd(int(d)))


def hyp1f1(a: float, b: float, z: float) -> float:
    """Plain series of 1F1."""
    return float(lib().or_hyp1f1(a, b, z))


def hyp1f2(a: float, b: float, c: float, z: float) -> float:
    """Plain series of 1F2 as defined at P:1153."""
    return float(lib().or_hyp1f2(a, b, c, z))


def F(kind: str, param: float, r, matern_p: int = 1) -> np.ndarray:
    """d-dimensional radial basis function F (Table 1; Matern P:1163).
    param: sigma (gaussian), ignored (negdist), ell with F=exp(-r/ell) (laplacian, R8), beta (matern)."""
    r = np.ascontiguousarray(np.atleast_1d(r), dtype=np.float64)
    out = np.empty_like(r)
    lib().or_F_vec(KIND[kind], float(param), int(matern_p), _ptr(r), _ptr(out), r.size)
    return out


def f(kind: str, param: float, d: int, r, matern_p: int = 1) -> np.ndarray:
    """1D counterpart f of F (Table 1, App. C), series in fp64; at d = 3 the closed form
    f = F + t F' of Cor 2.4 for the smooth kernels."""
    r = np.ascontiguousarray(np.atleast_1d(r), dtype=np.float64)
    out = np.empty_like(r)
    lib().or_f_vec(KIND[kind], float(param), int(matern_p), int(d), _ptr(r), _ptr(out), r.size)
    _check()
    return out


def f_series(kind: str, param: float, d: int, r, matern_p: int = 1) -> np.ndarray:
    """f by its defining series (Table 1 / App. C) at any d, bypassing the d = 3 closed form of Cor 2.4
     that ``f`` uses; for the pins comparing the two."""
    r = np.ascontiguousarray(np.atleast_1d(r), dtype=np.float64)
    out = np.empty_like(r)
    lib().or_f_series_vec(KIND[kind], float(param), int(matern_p), int(d), _ptr(r), _ptr(out), r.size)
    _check()
    return out


def splitmix64(z: int) -> int:
    return int(lib().or_splitmix64(ctypes.c_uint64(z & 0xFFFFFFFFFFFFFFFF)))


def round_bf16(v: float) -> float:
    return float(lib().or_round_bf16(float(v)))


def directions(P: int, d: int, seed: int, p0: int = 0, p1: Optional[int] = None):
    """(g, inv_norm): g (p1-p0) x d bf16-exact fp64 Gaussian draws, inv_norm = 1/||g_p|| (R1)."""
    p1 = P if p1 is None else p1
    g = np.empty((p1 - p0, d), dtype=np.float64)
    inv = np.empty(p1 - p0, dtype=np.float64)
    lib().or_directions(int(P), int(d), ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(p0), int(p1), _ptr(g), _ptr(inv))
    return g, inv


def unit_directions(P: int, d: int, seed: int, p0: int = 0, p1: Optional[int] = None) -> np.ndarray:
    """xi_p = g_p / ||g_p|| in fp64 (R1)."""
    g, inv = directions(P, d, seed, p0, p1)
    return g * inv[:, None]


def project(pts: np.ndarray, xi: np.ndarray) -> np.ndarray:
    """z[p][i] = <xi_p, pts_i> in fp64.  pts fp32 (n x d), xi fp64 (np x d)."""
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    n, d = pts.shape
    z = np.empty((xi.shape[0], n), dtype=np.float64)
    lib().or_project(_ptr(pts), n, d, _ptr(xi), xi.shape[0], _ptr(z))
    return z


def exact_sum(kind: str, param: float, x: np.ndarray, y: np.ndarray, w: np.ndarray,
              targets: Optional[np.ndarray] = None, matern_p: int = 1) -> np.ndarray:
    """(a) s_m = sum_n w_n F(||x_n - y_m||) in fp64, for m in targets (default all)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    tgt = np.arange(y.shape[0], dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    out = np.empty(tgt.size, dtype=np.float64)
    lib().or_exact_sum(KIND[kind], float(param), int(matern_p), x.shape[1], _ptr(x), x.shape[0], _ptr(y),
                       _ptr(tgt), tgt.size, _ptr(w), _ptr(out))
    return out


def sliced_sum(kind: str, param: float, x: np.ndarray, y: np.ndarray, w: np.ndarray, P: int, seed: int,
               targets: Optional[np.ndarray] = None, p0: int = 0, p1: Optional[int] = None,
               matern_p: int = 1, xi: Optional[np.ndarray] = None) -> np.ndarray:
    """(b) s_m = (1/P) sum_{p in [p0,p1)} sum_n w_n f(|<xi_p,x_n> - <xi_p,y_m>|)  (Alg. 1)
    with direct 1D sums on the seeded directions of DESIGN.md R1 (or ``xi`` if given)."""
    p1 = P if p1 is None else p1
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    d = x.shape[1]
    if xi is None:
        xi = unit_directions(P, d, seed, p0, p1)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    assert xi.shape == (p1 - p0, d)
    tgt = np.arange(y.shape[0], dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    out = np.empty(tgt.size, dtype=np.float64)
    lib().or_sliced_sum(KIND[kind], float(param), int(matern_p), d, _ptr(x), x.shape[0], _ptr(y), _ptr(tgt),
                        tgt.size, _ptr(w), int(P), int(p0), int(p1), _ptr(xi), _ptr(out))
    _check()
    return out


def sum_1d(kind: str, param: float, d: int, zx: np.ndarray, w: np.ndarray, zy: np.ndarray,
           matern_p: int = 1) -> np.ndarray:
    """t_m = sum_n w_n f(|zx_n - zy_m|) in fp64 on given 1D points."""
    zx = np.ascontiguousarray(zx, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    zy = np.ascontiguousarray(zy, dtype=np.float64)
    t = np.empty(zy.size, dtype=np.float64)
    lib().or_sum_1d(KIND[kind], float(param), int(matern_p), int(d), _ptr(zx), _ptr(w), zx.size, _ptr(zy), zy.size,
                    _ptr(t))
    _check()
    return t
