"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports every symbol
include/sks.h declares, validates arguments, fails loudly (SKS_ERR_CUDA) instead of falling back
when no device is present, reproduces the oracle's directions bit for bit, and its closed-form
torus coefficients (Lemma 2.5; R7/R7b) match independent numeric Fourier transforms /
torus reconstructions of the oracle's 1D counterparts."""
import ctypes
import math
import os
import re

import numpy as np
import pytest
from scipy import integrate

import oracle as O
from paper_2401_08260_b200 import _lib, build, sks_directions, sks_fourier_coeffs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return _lib.load()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sks.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sks_[a-z0-9_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"binding lacks {s}"
    assert L.sks_version().decode().startswith("sks")


def test_argument_validation(L):
    out = ctypes.c_size_t()
    k = _lib.kernel("gaussian", 1.0)
    assert L.sks_workspace_size(0, 10, 3, k, 8, 0, 8, None, ctypes.byref(out)) == _lib.SKS_ERR_INVALID
    assert L.sks_workspace_size(10, 10, 3, k, 8, 4, 2, None, ctypes.byref(out)) == _lib.SKS_ERR_INVALID
    assert L.sks_workspace_size(10, 10, 3, _lib.kernel("gaussian", -1.0), 8, 0, 8, None, ctypes.byref(out)) == \
        _lib.SKS_ERR_INVALID
    bad = _lib.sks_kernel(7, 0, 1.0)
    assert L.sks_workspace_size(10, 10, 3, bad, 8, 0, 8, None, ctypes.byref(out)) == _lib.SKS_ERR_UNSUPPORTED
    assert "unsupported" in L.sks_last_error().decode()
    assert L.sks_workspace_size(10, 10, 3, _lib.kernel("matern", 1.0, 9), 8, 0, 8, None,
                                ctypes.byref(out)) == _lib.SKS_ERR_UNSUPPORTED
    assert L.sks_workspace_size(100, 50, 3, k, 8, 0, 8, None, ctypes.byref(out)) == _lib.SKS_OK
    assert out.value > 0
    assert L.sks_workspace_size(100, 50, 3, k, 8, 0, 8, _lib.options(window_w=1), ctypes.byref(out)) == \
        _lib.SKS_ERR_INVALID


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_cpu_fallback_without_device(L):
    # compute entry points must fail with SKS_ERR_CUDA (never compute on the host)
    k = _lib.kernel("negdist", 1.0)
    fake = ctypes.c_void_p(1 << 20)
    st = L.sks_sum(fake, 10, fake, 10, 3, fake, k, 4, 1, 0, 4, fake, fake, 1 << 30, None, None)
    assert st == _lib.SKS_ERR_CUDA, (st, L.sks_last_error())
    x = np.zeros((10, 3), np.float32)
    s = np.zeros(10, np.float32)
    st = L.sks_sum_host(x.ctypes.data, 10, x.ctypes.data, 10, 3, s.ctypes.data, k, 4, 1, 0, 4, s.ctypes.data,
                        fake, 1 << 30, None, None)
    assert st == _lib.SKS_ERR_CUDA


@pytest.mark.parametrize("P,d,seed", [(64, 3, 101), (40, 50, 102), (7, 3072, 104), (9, 1, 5)])
def test_directions_bitwise_equal_to_oracle(P, d, seed):
    g, inv = sks_directions(P, d, seed)
    go, invo = O.directions(P, d, seed)
    np.testing.assert_array_equal(g.astype(np.float64), go)
    np.testing.assert_array_equal(inv, invo)
    g2, inv2 = sks_directions(P, d, seed, 2, 5)
    np.testing.assert_array_equal(g2, g[2:5])


def _numeric_fhat(fun, rho, xmax):
    # fhat(rho) = 2 int_0^inf f(x) cos(2 pi rho x) dx
    v, _ = integrate.quad(lambda x: fun(x) * math.cos(2 * math.pi * rho * x), 0.0, xmax, limit=800, epsabs=1e-13)
    return 2 * v


@pytest.mark.parametrize("d,sigma", [(1, 1.0), (3, 1.0), (3, 2.5)])
def test_gauss_coeffs_vs_numeric_ft(d, sigma):
    # Lemma 2.5 closed form (library) vs numeric FT of f (d=1: F; d=3: Cor 2.4 / oracle series)
    tau = 0.05
    ks = np.array([0, 1, 3, 6, 10, 15])
    c = sks_fourier_coeffs("gaussian", sigma, d, tau, 0, int(ks.max()))[ks]
    for k, ck in zip(ks, c):
        f = lambda x: float(O.f("gaussian", sigma, d, [x])[0])
        ref = tau * _numeric_fhat(f, tau * k, 14 * sigma)
        assert ck == pytest.approx(ref, abs=1e-10), (k, ck, ref)


@pytest.mark.parametrize("d,ell", [(1, 1.0), (3, 1.0), (3, 0.4)])
def test_laplace_fhat_vs_numeric_ft(d, ell):
    # R7: fhat_Lap(rho) = (2 c_d/alpha) s^{d-1} (1+s^2)^{-(d+1)/2}; the library coefficient minus the
    # companion term (alpha c_d/tau) hhat_k must equal tau * numeric FT of f (d=1: F; d=3: Cor 2.4)
    tau = 0.02
    alpha = 1.0 / ell
    A = O.cd(d) * alpha / tau
    for k in (1, 2, 5, 9):
        ck = sks_fourier_coeffs("laplacian", ell, d, tau, k, k)[0]
        f_part = ck + A / (2 * math.pi**2 * k * k)
        f = (lambda x: math.exp(-alpha * x)) if d == 1 else (lambda x: (1 - alpha * x) * math.exp(-alpha * x))
        ref = tau * _numeric_fhat(f, tau * k, 60 * ell)
        assert f_part == pytest.approx(ref, abs=1e-9), (k, f_part, ref)


@pytest.mark.parametrize("d,beta", [(1, 1.0), (3, 1.0)])
def test_matern_fhat_vs_numeric_ft(d, beta):
    tau = 0.03
    s3 = math.sqrt(3)
    f = (lambda x: (1 + s3 * x / beta) * math.exp(-s3 * x / beta)) if d == 1 else \
        (lambda x: (1 + s3 * x / beta - 3 * x * x / beta**2) * math.exp(-s3 * x / beta))
    for k in (0, 1, 4, 8, 20):
        ck = sks_fourier_coeffs("matern", beta, d, tau, k, k, matern_p=1)[0]
        ref = tau * _numeric_fhat(f, tau * k, 40 * beta)
        assert ck == pytest.approx(ref, abs=1e-10), (k, ck, ref)


@pytest.mark.parametrize("kind,scale,d", [("gaussian", 1.0, 50), ("laplacian", 2.0, 50), ("matern", 1.0, 10)])
def test_torus_reconstruction_high_d(kind, scale, d):
    # sum_k c_k e^{2 pi i k u} reproduces the periodised counterpart on the torus (R7 for the
    # Laplacian's smooth part psi = f(|u|/tau) + (alpha c_d/tau)(|u| - u^2)), checked against the oracle's f
    tau = 1.0 / (30.0 * scale)
    K = 6000
    c = sks_fourier_coeffs(kind, scale, d, tau, 0, K)
    us = np.linspace(0.0, 0.05, 11)   # |x| = u/tau <= 1.5 scale: where the oracle series is well conditioned
    kk = np.arange(1, K + 1)
    recon = np.array([c[0] + 2 * np.sum(c[1:] * np.cos(2 * np.pi * kk * u)) for u in us])
    ref = O.f(kind, scale, d, us / tau)
    if kind == "laplacian":
        ref = ref + (O.cd(d) / scale / tau) * (np.abs(us) - us**2)
    assert np.max(np.abs(recon - ref)) < 2e-6, np.max(np.abs(recon - ref))
