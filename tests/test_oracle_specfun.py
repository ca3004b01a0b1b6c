"""Pins for the oracle's special functions and 1D counterparts f (-m "not gpu").

Each test checks the oracle against something OTHER than its own formula: closed forms the
paper states for special cases (d=1: f=F by Thm 2.2; d=3: Cor 2.4), the S_d integral of
Prop 2.3 by independent quadrature (scipy), textbook hypergeometric identities, Monte-Carlo
slicing and the bound of Thm 2.7(i).
"""
import math

import numpy as np
import pytest
from scipy import integrate

import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore::scipy.integrate.IntegrationWarning")


def test_cd_closed_values():
    # c_d = sqrt(pi) Gamma((d+1)/2)/Gamma(d/2); Gamma(1/2)=sqrt(pi), Gamma(3/2)=sqrt(pi)/2
    assert O.cd(1) == pytest.approx(1.0, abs=1e-15)
    assert O.cd(3) == pytest.approx(2.0, abs=1e-15)
    assert O.cd(2) == pytest.approx(math.pi / 2, abs=1e-15)      # Gamma(3/2)/Gamma(1) * sqrt(pi)
    # Gamma(x+1/2)/Gamma(x) ~ sqrt(x) (1 - 1/(8x)): c_d ~ sqrt(pi d/2) (1 - 1/(4d))
    for d in (784, 3072):
        assert O.cd(d) == pytest.approx(math.sqrt(math.pi * d / 2) * (1 - 1 / (4 * d)), rel=1e-6)


@pytest.mark.parametrize("x", [0.0, 0.3, 1.0, 4.0, 10.0])
def test_hypergeometric_identities(x):
    assert O.hyp1f1(0.7, 0.7, -x) == pytest.approx(math.exp(-x), rel=1e-12, abs=1e-11)   # 1F1(c;c;-x)=e^-x (plain alternating series: abs. cancellation ~ e^x eps)
    assert O.hyp1f2(0.5, 0.5, 0.5, x * x / 4) == pytest.approx(math.cosh(x), rel=1e-13)   # sum x^2n/(2n)!
    if x > 0:
        assert O.hyp1f2(1.0, 1.0, 1.5, x * x / 4) == pytest.approx(math.sinh(x) / x, rel=1e-13)


R = np.linspace(0.0, 6.0, 61)


def test_d1_counterpart_equals_F():
    # Thm 2.2 with d=1: b_n = a_n, so f = F
    np.testing.assert_allclose(O.f("gaussian", 1.3, 1, R), np.exp(-R**2 / (2 * 1.3**2)), atol=1e-13)
    np.testing.assert_allclose(O.f("laplacian", 2.0, 1, R), np.exp(-R / 2.0), atol=1e-13)
    s3 = math.sqrt(3)
    np.testing.assert_allclose(O.f("matern", 1.5, 1, R, matern_p=1),
                               (1 + s3 * R / 1.5) * np.exp(-s3 * R / 1.5), atol=1e-11)
    np.testing.assert_allclose(O.f("negdist", 0, 1, R), -R, atol=1e-15)


def test_d3_cor24():
    # Cor 2.4: d=3 -> f(t) = F(t) + t F'(t).  The oracle evaluates this closed form at d = 3; pin it
    # against the defining series of Table 1 / App. C where the plain series is well
    # conditioned, and against the hand-differentiated forms
    s = 1.0
    np.testing.assert_allclose(O.f("gaussian", s, 3, R), (1 - R**2 / s**2) * np.exp(-R**2 / (2 * s**2)), atol=1e-12)
    a = 0.5
    np.testing.assert_allclose(O.f("laplacian", 1 / a, 3, R), (1 - a * R) * np.exp(-a * R), atol=1e-12)
    b, s3 = 1.0, math.sqrt(3)
    np.testing.assert_allclose(O.f("matern", b, 3, R, matern_p=1),
                               (1 + s3 * R / b - 3 * R**2 / b**2) * np.exp(-s3 * R / b), atol=1e-12)
    Rm = R[R <= 4.0]   # beyond, the plain alternating 1F2 series loses digits and the oracle's series refuses
    for kind, par, mp in [("gaussian", 1.0, 1), ("laplacian", 2.0, 1), ("matern", 1.0, 1), ("matern", 1.5, 2),
                          ("matern", 2.0, 0)]:
        np.testing.assert_allclose(O.f(kind, par, 3, Rm, matern_p=mp), O.f_series(kind, par, 3, Rm, matern_p=mp),
                                   atol=1e-9, err_msg=f"{kind} p={mp}")
    with pytest.raises(O.OracleConditioningError):
        O.f_series("matern", b, 3, [12.0], matern_p=1)
    np.testing.assert_allclose(O.f("negdist", 0, 3, R), -2 * R, atol=1e-14)


@pytest.mark.parametrize("kind,par,mp", [("gaussian", 1.0, 1), ("laplacian", 1.0, 1), ("matern", 1.0, 1),
                                         ("matern", 1.0, 2), ("matern", 0.7, 0)])
def test_d3_closed_form_by_S3_quadrature(kind, par, mp):
    # Prop 2.3 at d = 3: the weight (1-t^2)^0 and the constant 2 Gamma(3/2)/(sqrt(pi) Gamma(1)) = 1, so
    # F(s) = int_0^1 f(ts) dt.  Checked far beyond the series' conditioned range (s up to 20 beta)
    for s in (0.5, 2.0, 6.0, 12.0, 20.0):
        val, _ = integrate.quad(lambda t: float(O.f(kind, par, 3, [t * s], matern_p=mp)[0]), 0.0, 1.0, limit=400,
                                epsabs=1e-14, epsrel=1e-13)
        assert val == pytest.approx(float(O.F(kind, par, [s], matern_p=mp)[0]), abs=1e-12), (kind, mp, s)


def _Sd(fun, d, s):
    """Prop 2.3: F(s) = 2 Gamma(d/2)/(sqrt(pi) Gamma((d-1)/2)) int_0^1 f(ts)(1-t^2)^((d-3)/2) dt"""
    c = 2 * math.exp(math.lgamma(d / 2) - math.lgamma((d - 1) / 2)) / math.sqrt(math.pi)
    val, _ = integrate.quad(lambda t: fun(t * s) * (1 - t * t) ** ((d - 3) / 2), 0.0, 1.0, limit=400,
                            epsabs=1e-13, epsrel=1e-12)
    return c * val


def _Sd_highd(fun, d, s):
    """Prop 2.3 for large d: the weight (1-t^2)^((d-3)/2) <= exp(-40) beyond t = sqrt(80/(d-3)), so the
    integral is taken over [0, sqrt(80/(d-3))] with breakpoints at k/sqrt(d) (its width scale)."""
    c = 2 * math.exp(math.lgamma(d / 2) - math.lgamma((d - 1) / 2)) / math.sqrt(math.pi)
    t1 = math.sqrt(80.0 / (d - 3))
    pts = [k / math.sqrt(d) for k in range(1, int(t1 * math.sqrt(d)) + 1) if k / math.sqrt(d) < t1]
    val, _ = integrate.quad(lambda t: fun(t * s) * math.exp((d - 3) / 2 * math.log1p(-t * t)), 0.0, t1,
                            points=pts, limit=800, epsabs=1e-15, epsrel=1e-13)
    return c * val


# the BASELINE configs' own (kind, dimension, parameter): cfg5 Gaussian d=100, cfg3 Gaussian d=784 (sigma = median
# pairwise distance, R10/R11), cfg4 Laplacian d=3072 (ell = median pairwise distance); s spans the data's distances
HIGHD = [("gaussian", 100, 30.65994192636891, (5.0, 20.0, 30.0, 45.0, 60.0)),
         ("gaussian", 784, 11.025468358570834, (2.0, 5.0, 8.0, 11.0, 16.0)),
         ("laplacian", 3072, 22.62531764763029, (4.0, 15.0, 22.6, 30.0, 40.0))]


@pytest.mark.parametrize("kind,d,par,svals", HIGHD, ids=["cfg5", "cfg3", "cfg4"])
def test_Sd_quadrature_config_dimensions(kind, d, par, svals):
    # S_d f = F (Prop 2.3) at the dimensions and parameters the GPU parity tests run: pins the oracle's series for f
    # where a dropped term or a wrong index would show (d in 100 ... 3072)
    for s in svals:
        fs = lambda r: float(O.f(kind, par, d, [r])[0])
        # (the Laplacian's f has a |r| kink at 0 that the quadrature resolves to ~1e-12)
        tol = 2e-12 if kind == "laplacian" else 1e-12
        assert _Sd_highd(fs, d, s) == pytest.approx(float(O.F(kind, par, [s])[0]), abs=tol), (kind, d, s)


@pytest.mark.parametrize("d", [2, 5, 10, 50])
def test_Sd_quadrature_gaussian(d):
    sigma = 1.0 if d <= 10 else 3.0
    for s in (0.3, 1.0, 2.0, 4.0):
        fs = lambda r: float(O.f("gaussian", sigma, d, [r])[0])
        assert _Sd(fs, d, s) == pytest.approx(math.exp(-s * s / (2 * sigma * sigma)), abs=1e-8)


@pytest.mark.parametrize("d", [2, 5, 10, 50])
def test_Sd_quadrature_laplacian(d):
    ell = 2.0 if d <= 10 else 8.0
    for s in (0.3, 1.0, 2.0, 4.0):
        fs = lambda r: float(O.f("laplacian", ell, d, [r])[0])
        assert _Sd(fs, d, s) == pytest.approx(math.exp(-s / ell), abs=1e-8)


@pytest.mark.parametrize("d", [2, 5, 10, 50])
def test_Sd_quadrature_matern(d):
    beta = 1.0 if d <= 10 else 4.0
    for s in (0.3, 1.0, 2.0, 3.0):
        fs = lambda r: float(O.f("matern", beta, d, [r], matern_p=1)[0])
        assert _Sd(fs, d, s) == pytest.approx(float(O.F("matern", beta, [s], matern_p=1)[0]), abs=1e-8)


@pytest.mark.parametrize("d", [5, 10])
def test_Sd_quadrature_matern_p2(d):
    beta = 1.0
    for s in (0.5, 1.5):
        fs = lambda r: float(O.f("matern", beta, d, [r], matern_p=2)[0])
        assert _Sd(fs, d, s) == pytest.approx(float(O.F("matern", beta, [s], matern_p=2)[0]), abs=1e-8)


def test_matern_F_halfint_textbook():
    # P:1163 at p=0 is the Laplacian; p=1,2 the textbook nu=3/2, 5/2 Matern forms
    r = np.linspace(0, 5, 11)
    np.testing.assert_allclose(O.F("matern", 2.0, r, matern_p=0), np.exp(-r / 2.0), rtol=1e-14)
    q = math.sqrt(3) * r
    np.testing.assert_allclose(O.F("matern", 1.0, r, matern_p=1), (1 + q) * np.exp(-q), rtol=1e-14)
    q = math.sqrt(5) * r
    np.testing.assert_allclose(O.F("matern", 1.0, r, matern_p=2), (1 + q + q * q / 3) * np.exp(-q), rtol=1e-13)


@pytest.mark.parametrize("d", [3, 50, 784])
def test_gauss_counterpart_bounded(d):
    # Thm 2.7(i): |f_sigma| <= 1
    sigma = 1.0 if d < 100 else 11.0
    r = np.linspace(0, 6 * sigma / math.sqrt(max(d, 1) / 3), 200) if d > 3 else np.linspace(0, 8, 200)
    v = O.f("gaussian", sigma, d, r)
    assert np.all(np.abs(v) <= 1 + 1e-12)
    assert v[0] == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("kind,param,d", [("gaussian", 1.0, 10), ("laplacian", 2.0, 10), ("matern", 1.0, 6)])
def test_monte_carlo_slicing(kind, param, d):
    # Eq. (sliced kernel) P:54-56 / Prop 2.3: E_xi f(|<xi,z>|) = F(||z||), MC over the oracle's directions
    rng = np.random.default_rng(5)
    xi = O.unit_directions(200_000, d, seed=77)
    for _ in range(3):
        z = rng.standard_normal(d)
        z *= 1.2 / np.linalg.norm(z)
        proj = np.abs(xi @ z)
        vals = O.f(kind, param, d, proj)
        est, se = vals.mean(), vals.std() / math.sqrt(vals.size)
        F = float(O.F(kind, param, [np.linalg.norm(z)])[0])
        assert abs(est - F) < 5 * se + 1e-12, (est, F, se)
