"""paper_2401_08260_b200 -- sliced fast kernel summation (arXiv 2401.08260) on B200.

Thin Python binding of libsks.so (include/sks.h) with the same names.  PyTorch supplies device
memory and streams only; every step of the hot path runs in the library's sm_100a kernels.
There is no CPU fallback: without the built library or a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from ._lib import SKSError, check, kernel, options  # noqa: F401

__all__ = ["sks_workspace_size", "sks_sum", "sks_sum_host", "sks_workspace_size_host", "sks_directions",
           "sks_project", "sks_sum_1d", "sks_workspace_size_1d", "sks_fourier_coeffs", "sks_last_plan", "sks_sync_status",
           "sks_version", "sks_release_caches", "sks_profile_enable", "sks_profile_read", "SKSError"]


def _torch():
    import torch
    return torch


ENGINES = {"auto": 0, "nfft": 1, "ndft": 2}
PROJECTIONS = {"auto": 0, "bf16x3": 1, "tf32x2": 2, "fp16x2": 3}


def _opts(eps=0.0, window_w=0, oversample=0, slice_batch=0, engine="auto", projection="auto", async_=False,
          graph=False, deterministic=False, exchange=None):
    e = ENGINES[engine] if isinstance(engine, str) else int(engine)
    pj = PROJECTIONS[projection] if isinstance(projection, str) else int(projection)
    if not (eps or window_w or oversample or slice_batch or e or pj or async_ or graph or deterministic
            or exchange is not None):
        return None
    return options(eps, window_w, oversample, slice_batch, e, pj, int(bool(async_)), int(bool(graph)),
                   int(bool(deterministic)), exchange)


def _stream_ptr(stream) -> Optional[int]:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _alloc_workspace(nbytes: int, device):
    torch = _torch()
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def sks_version() -> str:
    return _lib.load().sks_version().decode()


def sks_release_caches() -> None:
    """Free the library's device caches (directions, planner tables, CUDA graphs); include/sks.h."""
    check(_lib.load().sks_release_caches())


def sks_workspace_size(N: int, M: int, d: int, kind: str, scale: float, P: int, p_begin: int = 0,
                       p_end: Optional[int] = None, matern_p: int = 1, **opts) -> int:
    L = _lib.load()
    out = ctypes.c_size_t(0)
    check(L.sks_workspace_size(N, M, d, kernel(kind, scale, matern_p), P, p_begin, P if p_end is None else p_end,
                               _opts(**opts), ctypes.byref(out)))
    return int(out.value)


def sks_workspace_size_host(N: int, M: int, d: int, kind: str, scale: float, P: int, p_begin: int = 0,
                            p_end: Optional[int] = None, matern_p: int = 1, **opts) -> int:
    L = _lib.load()
    out = ctypes.c_size_t(0)
    check(L.sks_workspace_size_host(N, M, d, kernel(kind, scale, matern_p), P, p_begin,
                                    P if p_end is None else p_end, _opts(**opts), ctypes.byref(out)))
    return int(out.value)


def sks_sum(x, y, w, kind: str, scale: float, P: int, seed: int, p_begin: int = 0, p_end: Optional[int] = None,
            matern_p: int = 1, out=None, workspace=None, stream=None, **opts):
    """s (M,) fp32 on x.device = (1/P) sum_{p in [p_begin,p_end)} t_{m,p}  (Alg. 1).
    x (N,d), y (M,d), w (N,) contiguous fp32 CUDA tensors."""
    torch = _torch()
    L = _lib.load()
    assert x.is_cuda and y.is_cuda and w.is_cuda, "sks_sum takes CUDA tensors (no CPU fallback)"
    assert x.dtype == y.dtype == w.dtype == torch.float32
    x, y, w = x.contiguous(), y.contiguous(), w.contiguous()
    N, d = x.shape
    M = y.shape[0]
    p_end = P if p_end is None else p_end
    o = _opts(**opts)
    if workspace is None:
        workspace = _alloc_workspace(sks_workspace_size(N, M, d, kind, scale, P, p_begin, p_end, matern_p, **opts),
                                     x.device)
    s = out if out is not None else torch.empty(M, dtype=torch.float32, device=x.device)
    check(L.sks_sum(x.data_ptr(), N, y.data_ptr(), M, d, w.data_ptr(), kernel(kind, scale, matern_p), P,
                    ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), p_begin, p_end, s.data_ptr(), workspace.data_ptr(),
                    workspace.numel(), o, _stream_ptr(stream)))
    return s


def sks_sum_host(x: np.ndarray, y: np.ndarray, w: np.ndarray, kind: str, scale: float, P: int, seed: int,
                 p_begin: int = 0, p_end: Optional[int] = None, matern_p: int = 1, out: Optional[np.ndarray] = None,
                 workspace=None, stream=None, **opts) -> np.ndarray:
    """Same as sks_sum from HOST arrays (copied in/out inside the call).  Pinned host tensors'
    numpy views may be passed for full copy bandwidth."""
    L = _lib.load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    N, d = x.shape
    M = y.shape[0]
    p_end = P if p_end is None else p_end
    if workspace is None:
        workspace = _alloc_workspace(
            sks_workspace_size_host(N, M, d, kind, scale, P, p_begin, p_end, matern_p, **opts), "cuda")
    s = out if out is not None else np.empty(M, dtype=np.float32)
    check(L.sks_sum_host(x.ctypes.data, N, y.ctypes.data, M, d, w.ctypes.data, kernel(kind, scale, matern_p), P,
                         ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), p_begin, p_end, s.ctypes.data,
                         workspace.data_ptr(), workspace.numel(), _opts(**opts), _stream_ptr(stream)))
    return s


def sks_directions(P: int, d: int, seed: int, p_begin: int = 0, p_end: Optional[int] = None):
    """(g, inv_norm): g (np, d) fp32 bf16-exact draws, inv_norm (np,) fp64 (R1).  Host only."""
    L = _lib.load()
    p_end = P if p_end is None else p_end
    g = np.empty((p_end - p_begin, d), dtype=np.float32)
    inv = np.empty(p_end - p_begin, dtype=np.float64)
    check(L.sks_directions(P, d, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), p_begin, p_end, g.ctypes.data,
                           inv.ctypes.data))
    return g, inv


def sks_project(pts, P: int, seed: int, p_begin: int = 0, p_end: Optional[int] = None, stream=None,
                projection: str = "auto"):
    """z (np, n) fp32 = <xi_p, pts_i> (row a1) for CUDA pts (n, d)."""
    torch = _torch()
    L = _lib.load()
    pts = pts.contiguous()
    n, d = pts.shape
    p_end = P if p_end is None else p_end
    z = torch.empty((p_end - p_begin, n), dtype=torch.float32, device=pts.device)
    check(L.sks_project(pts.data_ptr(), n, d, P, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), p_begin, p_end,
                        z.data_ptr(), _opts(projection=projection), _stream_ptr(stream)))
    return z


def sks_workspace_size_1d(N: int, M: int, d: int, kind: str, scale: float, n_slices: int, matern_p: int = 1,
                          **opts) -> int:
    L = _lib.load()
    out = ctypes.c_size_t(0)
    check(L.sks_workspace_size_1d(N, M, d, kernel(kind, scale, matern_p), n_slices, _opts(**opts), ctypes.byref(out)))
    return int(out.value)


def sks_sum_1d(zx, zy, w, d: int, kind: str, scale: float, matern_p: int = 1, workspace=None, stream=None, **opts):
    """t (S, M): per-slice 1D sums t[q, m] = sum_n w_n f(|zx[q,n] - zy[q,m]|) (rows a2-a7) on CUDA tensors."""
    torch = _torch()
    L = _lib.load()
    zx, zy, w = zx.contiguous(), zy.contiguous(), w.contiguous()
    S, N = zx.shape
    M = zy.shape[1]
    if workspace is None:
        workspace = _alloc_workspace(sks_workspace_size_1d(N, M, d, kind, scale, S, matern_p, **opts), zx.device)
    t = torch.empty((S, M), dtype=torch.float32, device=zx.device)
    check(L.sks_sum_1d(zx.data_ptr(), zy.data_ptr(), w.data_ptr(), N, M, S, d, kernel(kind, scale, matern_p),
                       t.data_ptr(), workspace.data_ptr(), workspace.numel(), _opts(**opts), _stream_ptr(stream)))
    return t


def sks_fourier_coeffs(kind: str, scale: float, d: int, tau: float, k0: int, k1: int, matern_p: int = 1) -> np.ndarray:
    """Torus coefficients c_k, k in [k0, k1], used by the planner (host only)."""
    L = _lib.load()
    out = np.empty(k1 - k0 + 1, dtype=np.float64)
    check(L.sks_fourier_coeffs(kernel(kind, scale, matern_p), d, float(tau), k0, k1, out.ctypes.data))
    return out


def sks_profile_enable(enable: bool = True) -> None:
    check(_lib.load().sks_profile_enable(1 if enable else 0))


def sks_profile_read() -> dict:
    """{slot: (ms, launches)} accumulated since the last read (blocks on the recorded events)."""
    L = _lib.load()
    ms = np.zeros(16, np.float64)
    cnt = np.zeros(16, np.int64)
    check(L.sks_profile_read(ms.ctypes.data, cnt.ctypes.data, 16))
    names = L.sks_profile_names().decode().split(",")
    return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(names)}


def sks_sync_status(workspace, stream=None) -> None:
    """Synchronise the stream and raise SKSError if the last call on `workspace` (async / graph) failed."""
    check(_lib.load().sks_sync_status(workspace.data_ptr(), _stream_ptr(stream)))


def sks_last_plan() -> dict:
    L = _lib.load()
    info = _lib.sks_plan_info()
    check(L.sks_last_plan(ctypes.byref(info)))
    return info.as_dict()
