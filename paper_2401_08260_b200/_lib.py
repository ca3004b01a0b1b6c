"""ctypes binding of libsks.so (include/sks.h).  Argument marshalling only: every step of the hot
path runs in the library's sm_100a kernels.  There is no fallback: if the library (or a CUDA device
for the compute calls) is missing, calls raise."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SKS_LIB selects another build of the same library (the bounds-checked libsks_checked.so of build.py --checked)
LIB_PATH = os.environ.get("SKS_LIB") or os.path.join(HERE, "libsks.so")

SKS_OK, SKS_ERR_INVALID, SKS_ERR_UNSUPPORTED, SKS_ERR_CUDA, SKS_ERR_WORKSPACE, SKS_ERR_NONFINITE = range(6)
STATUS_NAMES = {0: "SKS_OK", 1: "SKS_ERR_INVALID", 2: "SKS_ERR_UNSUPPORTED", 3: "SKS_ERR_CUDA",
                4: "SKS_ERR_WORKSPACE", 5: "SKS_ERR_NONFINITE"}
KINDS = {"gaussian": 0, "negdist": 1, "laplacian": 2, "matern": 3}


class sks_kernel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("matern_p", ctypes.c_int32), ("scale", ctypes.c_double)]


class sks_options(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("window_w", ctypes.c_int32), ("oversample", ctypes.c_int32),
                ("slice_batch", ctypes.c_int32), ("engine", ctypes.c_int32), ("projection", ctypes.c_int32),
                ("async_", ctypes.c_int32), ("deterministic", ctypes.c_int32), ("graph", ctypes.c_int32),
                ("exchange", ctypes.c_void_p), ("exchange_user", ctypes.c_void_p)]


# int (*sks_exchange_fn)(void* user, int32_t op, void* dev_ptr, size_t count, void* stream)   (include/sks.h)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p)
XCHG_BCAST_F64, XCHG_MAX_I32, XCHG_SUM_F32 = 0, 1, 2


class sks_plan_info(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("n_grid", ctypes.c_int32), ("k_max", ctypes.c_int32),
                ("band_lo_min", ctypes.c_int32), ("window_w", ctypes.c_int32), ("spread_cells", ctypes.c_int32),
                ("n_buckets", ctypes.c_int32), ("slice_batch", ctypes.c_int32), ("n_batches", ctypes.c_int32),
                ("launches", ctypes.c_int32), ("tau_min", ctypes.c_double), ("tau_max", ctypes.c_double),
                ("engine", ctypes.c_int32), ("band_width", ctypes.c_int32),
                ("proj_mode", ctypes.c_int32), ("fused", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# every symbol include/sks.h declares, with its ctypes signature
_i32, _i64, _u64, _vp, _sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
_K, _O = sks_kernel, ctypes.POINTER(sks_options)
SIGNATURES = {
    "sks_workspace_size": (_i32, [_i64, _i64, _i32, _K, _i32, _i32, _i32, _O, ctypes.POINTER(_sz)]),
    "sks_sum": (_i32, [_vp, _i64, _vp, _i64, _i32, _vp, _K, _i32, _u64, _i32, _i32, _vp, _vp, _sz, _O, _vp]),
    "sks_workspace_size_host": (_i32, [_i64, _i64, _i32, _K, _i32, _i32, _i32, _O, ctypes.POINTER(_sz)]),
    "sks_sum_host": (_i32, [_vp, _i64, _vp, _i64, _i32, _vp, _K, _i32, _u64, _i32, _i32, _vp, _vp, _sz, _O, _vp]),
    "sks_directions": (_i32, [_i32, _i32, _u64, _i32, _i32, _vp, _vp]),
    "sks_project": (_i32, [_vp, _i64, _i32, _i32, _u64, _i32, _i32, _vp, _O, _vp]),
    "sks_workspace_size_1d": (_i32, [_i64, _i64, _i32, _K, _i32, _O, ctypes.POINTER(_sz)]),
    "sks_sum_1d": (_i32, [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _K, _vp, _vp, _sz, _O, _vp]),
    "sks_fourier_coeffs": (_i32, [_K, _i32, ctypes.c_double, _i32, _i32, _vp]),
    "sks_last_plan": (_i32, [ctypes.POINTER(sks_plan_info)]),
    "sks_sync_status": (_i32, [_vp, _vp]),
    "sks_profile_enable": (_i32, [_i32]),
    "sks_profile_read": (_i32, [_vp, _vp, _i32]),
    "sks_profile_names": (ctypes.c_char_p, []),
    "sks_release_caches": (_i32, []),
    "sks_last_error": (ctypes.c_char_p, []),
    "sks_version": (ctypes.c_char_p, []),
}

_lib = None


class SKSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def load() -> ctypes.CDLL:
    """Load libsks.so (build it first with paper_2401_08260_b200.build.build()).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run paper_2401_08260_b200.build.build() (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != SKS_OK:
        raise SKSError(status, load().sks_last_error().decode())


def kernel(kind: str, scale: float = 1.0, matern_p: int = 1) -> sks_kernel:
    return sks_kernel(KINDS[kind], int(matern_p), float(scale))


def options(eps: float = 0.0, window_w: int = 0, oversample: int = 0, slice_batch: int = 0, engine: int = 0,
            projection: int = 0, async_: int = 0, graph: int = 0, deterministic: int = 0, exchange=None):
    """exchange: an EXCHANGE_FN instance (kept alive by the caller for the duration of the call) or None"""
    fn = ctypes.cast(exchange, ctypes.c_void_p) if exchange is not None else None
    return ctypes.pointer(sks_options(float(eps), int(window_w), int(oversample), int(slice_batch), int(engine),
                                      int(projection), int(async_), int(deterministic), int(graph), fn, None))
