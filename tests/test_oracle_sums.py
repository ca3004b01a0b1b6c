"""Pins for the oracle's sums, projections and directions (-m "not gpu").

Hand-computed tiny cases (tests/golden/tiny_sums.json, each with its source), the exactness of
slicing in d=1, translation invariance, the closed-form identity E|<xi,z>| = ||z||/c_d,
the SplitMix64 published test vector, bf16 round-to-nearest-even cases, and the slicing-error
rate O(P^{-1/2}) of Prop 2.6 / Thm 2.7.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tiny_sums.json")))


@pytest.mark.parametrize("case", GOLD["negdist_1d"], ids=lambda c: c["source"][:24])
def test_negdist_1d_golden(case):
    t = O.sum_1d("negdist", 0.0, case["d"], np.array(case["x"]), np.array(case["w"]), np.array(case["y"]))
    np.testing.assert_allclose(t, case["t"], atol=1e-14)


def test_exact_sum_golden():
    c = GOLD["exact_dd"][0]
    x, y, w = np.array(c["x"]), np.array(c["y"]), np.array(c["w"])
    assert O.exact_sum("negdist", 0, x, y, w)[0] == pytest.approx(c["negdist"], abs=1e-14)
    assert O.exact_sum("gaussian", 5.0, x, y, w)[0] == pytest.approx(c["gaussian_sigma5"], abs=1e-14)
    assert O.exact_sum("laplacian", 5.0, x, y, w)[0] == pytest.approx(c["laplacian_ell5"], abs=1e-14)
    assert O.exact_sum("matern", 5.0, x, y, w, matern_p=1)[0] == pytest.approx(c["matern_p1_beta5"], abs=1e-14)


@pytest.mark.parametrize("kind,param", [("gaussian", 0.8), ("negdist", 0.0), ("laplacian", 1.5), ("matern", 1.0)])
def test_d1_slicing_is_exact(kind, param):
    # S^0 = {+1,-1}: |<xi,x-y>| = |x-y|, and f = F in d=1, so (b) == (a)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((50, 1)).astype(np.float32)
    y = rng.standard_normal((20, 1)).astype(np.float32)
    w = rng.uniform(-1, 1, 50).astype(np.float32)
    a = O.exact_sum(kind, param, x, y, w)
    b = O.sliced_sum(kind, param, x, y, w, P=7, seed=3)
    np.testing.assert_allclose(b, a, atol=1e-12)


def test_translation_invariance_negdist():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((40, 5)).astype(np.float32)
    y = rng.standard_normal((10, 5)).astype(np.float32)
    w = rng.random(40).astype(np.float32)
    shift = np.float32(4.0)
    b0 = O.sliced_sum("negdist", 0, x, y, w, P=16, seed=9)
    b1 = O.sliced_sum("negdist", 0, x + shift, y + shift, w, P=16, seed=9)
    np.testing.assert_allclose(b1, b0, atol=1e-5)   # fp32 rounding of the shifted inputs


def test_projection_basics():
    rng = np.random.default_rng(3)
    pts = rng.standard_normal((30, 6)).astype(np.float32)
    e1 = np.zeros((1, 6))
    e1[0, 0] = 1.0
    np.testing.assert_array_equal(O.project(pts, e1)[0], pts[:, 0].astype(np.float64))
    xi = O.unit_directions(8, 6, seed=4)
    z = O.project(pts, xi)
    assert np.all(np.abs(z) <= np.linalg.norm(pts.astype(np.float64), axis=1)[None, :] + 1e-12)   # Cauchy-Schwarz


def test_splitmix64_vector():
    # Published first output of SplitMix64 started from state 0 (Vigna's reference splitmix64.c)
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF


def test_bf16_round_nearest_even():
    assert O.round_bf16(1.0 + 2**-8) == 1.0                 # tie -> even (mantissa 0)
    assert O.round_bf16(1.0 + 3 * 2**-8) == 1.0 + 2**-6     # tie -> even (mantissa 2)
    assert O.round_bf16(1.0 + 2**-8 + 2**-20) == 1.0 + 2**-7
    assert O.round_bf16(-1.5) == -1.5


def test_directions_properties():
    g, inv = O.directions(64, 37, seed=11)
    # bf16-exact: every component has at most 8 significant bits
    m, e = np.frexp(g)
    assert np.all(m * 256 == np.round(m * 256))
    xi = g * inv[:, None]
    np.testing.assert_allclose(np.linalg.norm(xi, axis=1), 1.0, atol=1e-15)
    # sub-range reproduces the full draw (one substream per slice)
    g2, inv2 = O.directions(64, 37, seed=11, p0=20, p1=40)
    np.testing.assert_array_equal(g2, g[20:40])
    np.testing.assert_array_equal(inv2, inv[20:40])
    # d = 1 -> xi = +-1
    xi1 = O.unit_directions(100, 1, seed=5)
    np.testing.assert_allclose(np.abs(xi1), 1.0, atol=2e-16)
    # isotropy: mean of many directions ~ 0 (CLT: ||mean|| ~ sqrt(1/P))
    xim = O.unit_directions(100_000, 10, seed=6).mean(axis=0)
    assert np.linalg.norm(xim) < 0.02


def test_negdist_identity_E_abs_proj():
    # E|<xi,z>| = ||z|| Gamma(d/2)/(sqrt(pi) Gamma((d+1)/2)) = ||z||/c_d (P:205 / Thm 2.2 with a_1=-1):
    # sliced negdist of one pair = -c_d E|<xi,x-y>| = -||x-y||
    for d in (3, 50):
        rng = np.random.default_rng(d)
        x = rng.standard_normal((1, d)).astype(np.float32)
        y = rng.standard_normal((1, d)).astype(np.float32)
        P = 200_000
        xi = O.unit_directions(P, d, seed=8)
        vals = -O.cd(d) * np.abs(xi @ (x[0].astype(np.float64) - y[0].astype(np.float64)))
        se = vals.std() / math.sqrt(P)
        b = O.sliced_sum("negdist", 0, x, y, np.ones(1, np.float32), P=P, seed=8)[0]
        assert b == pytest.approx(vals.mean(), rel=1e-10)
        r = float(np.linalg.norm(x[0].astype(np.float64) - y[0].astype(np.float64)))
        assert abs(b + r) < 5 * se


@pytest.mark.parametrize("kind,param,d", [("negdist", 0.0, 10), ("gaussian", 1.0, 3)])
def test_slicing_error_rate(kind, param, d):
    # Prop 2.6 / Thm 2.7: E|est - K| = O(P^{-1/2}); fitted log-log slope of the per-summand error
    rng = np.random.default_rng(10)
    x = rng.standard_normal((60, d)).astype(np.float32)
    y = rng.standard_normal((30, d)).astype(np.float32)
    w = rng.random(60).astype(np.float32)
    a = O.exact_sum(kind, param, x, y, w)
    Ps = [16, 64, 256, 1024]
    errs = []
    for P in Ps:
        e = [np.abs(O.sliced_sum(kind, param, x, y, w, P=P, seed=100 + rep) - a).mean() for rep in range(6)]
        errs.append(np.mean(e) / np.abs(w).sum())
    slope = np.polyfit(np.log(Ps), np.log(errs), 1)[0]
    assert -0.65 < slope < -0.35, (slope, errs)
