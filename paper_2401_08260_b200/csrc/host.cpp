// host.cpp -- host-side runtime of libsks: directions (R1) and the torus / NFFT planner
// (Sec. 3.1; readings R3-R7b in DESIGN.md).  Pure C++17, fp64, no CUDA.
// This file shares no code with oracle/ (the oracle is test infrastructure only).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "host.h"

namespace sks {

static const double kPi = 3.14159265358979323846;

// ------------------------------------------------------------------ directions (R1)
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline float to_bf16_rne(double v) {
  float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

void make_directions(int P, int d, uint64_t seed, int p0, int p1, float* g, double* inv_norm) {
  (void)P;
  for (int p = p0; p < p1; ++p) {
    const uint64_t key = mix64(seed ^ mix64(static_cast<uint64_t>(p)));
    float* gp = g + static_cast<int64_t>(p - p0) * d;
    for (int q = 0; 2 * q < d; ++q) {
      const uint64_t a = mix64(key + 2ULL * q), b = mix64(key + 2ULL * q + 1ULL);
      const double u1 = (static_cast<double>(a >> 11) + 0.5) * 0x1.0p-53;
      const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
      const double rad = std::sqrt(-2.0 * std::log(u1)), ang = 2.0 * kPi * u2;
      gp[2 * q] = to_bf16_rne(rad * std::cos(ang));
      if (2 * q + 1 < d) gp[2 * q + 1] = to_bf16_rne(rad * std::sin(ang));
    }
    double ss = 0.0;
    for (int j = 0; j < d; ++j) ss += static_cast<double>(gp[j]) * gp[j];
    inv_norm[p - p0] = 1.0 / std::sqrt(ss);
  }
}

// ------------------------------------------------------------------ kernel model
double cd(int d) {
  thread_local int last_d = -1;
  thread_local double last_v = 0.0;
  if (d != last_d) {
    last_v = std::sqrt(kPi) * std::exp(std::lgamma(0.5 * (d + 1)) - std::lgamma(0.5 * d));
    last_d = d;
  }
  return last_v;
}

// unit-scale fhat (scale = 1)
double fhat1(const KernelModel& k, double rho) {
  rho = std::fabs(rho);
  const int d = k.d;
  switch (k.kind) {
    case 0: {  // Gaussian, Lemma 2.5: d pi e^{-2 pi^2 w^2} (2 pi^2 w^2)^{(d-1)/2} / (sqrt2 Gamma(d/2+1))
      if (rho == 0.0) return d == 1 ? std::sqrt(2.0 * kPi) : 0.0;
      const double a = 2.0 * kPi * kPi * rho * rho;
      return std::exp(std::log(d * kPi / std::sqrt(2.0)) - std::lgamma(0.5 * d + 1.0) - a + 0.5 * (d - 1) * std::log(a));
    }
    case 2: {  // Laplacian (alpha = 1), R7: 2 c_d s^{d-1} (1+s^2)^{-(d+1)/2}, s = 2 pi rho
      const double s = 2.0 * kPi * rho;
      if (s == 0.0) return d == 1 ? 2.0 : 0.0;
      return 2.0 * cd(d) * std::exp((d - 1) * std::log(s) - 0.5 * (d + 1) * std::log1p(s * s));
    }
    case 3: {  // Matern nu = p+1/2, beta = 1, R7b: (pi^{d/2}/Gamma(d/2)) rho^{d-1} Khat_d(rho)
      const double nu = k.matern_p + 0.5;
      const double logK = d * std::log(2.0) + 0.5 * d * std::log(kPi) + std::lgamma(nu + 0.5 * d) + nu * std::log(2.0 * nu) -
                          std::lgamma(nu) - (nu + 0.5 * d) * std::log(2.0 * nu + 4.0 * kPi * kPi * rho * rho);
      if (rho == 0.0) return d == 1 ? std::exp(0.5 * std::log(kPi) - std::lgamma(0.5) + logK) : 0.0;
      return std::exp(0.5 * d * std::log(kPi) - std::lgamma(0.5 * d) + (d - 1) * std::log(rho) + logK);
    }
  }
  return 0.0;
}

double torus_coeff(const KernelModel& k, double tau, int64_t kk) {
  // f(x) = f1(x/scale)  =>  fhat(rho) = scale fhat1(scale rho); periodised on 1/tau: c_k = tau fhat(tau k)
  double c = tau * k.scale * fhat1(k, k.scale * tau * static_cast<double>(kk));
  if (k.kind == 2) {  // Laplacian smooth part psi = f(|u|/tau) + (alpha c_d/tau) h(u), h = |u| - u^2 (R7)
    const double A = cd(k.d) / (k.scale * tau);
    c += (kk == 0) ? A / 6.0 : -A / (2.0 * kPi * kPi * static_cast<double>(kk) * static_cast<double>(kk));
  }
  return c;
}

// ------------------------------------------------------------------ decay radius (R3)
// f1(x) = 2 int_0^inf fhat1(r) cos(2 pi r x) dr   (fhat1 even, real).  Laplacian: the |x| kink gives a
// rho^-2 tail, so we subtract c_d * FT[e^{-|x|}] = 2 c_d/(1+4 pi^2 rho^2) and add c_d e^{-x} back.
static double integrand(const KernelModel& k, double r) {
  double v = fhat1(k, r);
  if (k.kind == 2) v -= 2.0 * cd(k.d) / (1.0 + 4.0 * kPi * kPi * r * r);
  return v;
}

static double unit_decay_radius(const KernelModel& k, double eps) {
  // rho range: up to where the remaining tail of |integrand| is below 1e-3 eps
  double peak = 0.0, rpk = 0.0;
  for (double r = 0.0; r < 1e4; r += 0.01) {
    double v = std::fabs(integrand(k, r));
    if (v > peak) { peak = v; rpk = r; }
    if (r > 2.0 * rpk + 5.0 && v < 1e-30) break;
  }
  double rmax = std::max(1.0, rpk);
  for (;;) {
    const double v = std::fabs(integrand(k, rmax));
    // tails: Gaussian super-exponential; Matern ~ r^{-2nu-1}; Laplacian (after subtraction) ~ r^{-4}
    const double tail = (k.kind == 0) ? v : v * rmax;   // crude integral bound for algebraic tails
    if (rmax > rpk && tail < 1e-3 * eps) break;
    rmax *= 1.25;
    if (rmax > 1e6) break;
  }
  double xmax = 16.0;
  for (int it = 0; it < 12; ++it) {
    const int nx = 400;
    const double dx = xmax / nx;
    const double h = 1.0 / (6.0 * xmax);
    const int64_t nr = static_cast<int64_t>(std::ceil(rmax / h)) + 1;
    std::vector<double> g(nr);
    for (int64_t i = 0; i < nr; ++i) g[i] = integrand(k, i * h) * (i == 0 ? 0.5 : 1.0);
    double last = 0.0;
    for (int ix = nx; ix >= 0; --ix) {
      const double x = ix * dx;
      // sum_i g_i cos(2 pi i h x) by complex rotation, re-anchored every 512 steps
      double s = 0.0;
      const double th = 2.0 * kPi * h * x;
      const double cr = std::cos(th), sr = std::sin(th);
      double c = 1.0, sn = 0.0;
      for (int64_t i = 0; i < nr; ++i) {
        if ((i & 511) == 0) { c = std::cos(th * i); sn = std::sin(th * i); }
        s += g[i] * c;
        const double c2 = c * cr - sn * sr;
        sn = sn * cr + c * sr;
        c = c2;
      }
      double f = 2.0 * h * s;
      if (k.kind == 2) f += cd(k.d) * std::exp(-x);
      if (std::fabs(f) > eps) { last = x; break; }
    }
    if (last < 0.75 * xmax) return last + 2.0 * dx;
    xmax *= 2.0;
  }
  return xmax;
}

double decay_radius(const KernelModel& k, double eps) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, double>, double> cache;
  const auto key = std::make_tuple(k.kind, k.kind == 3 ? k.matern_p : 0, k.d, eps);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second * k.scale;
  }
  KernelModel unit = k;
  unit.scale = 1.0;
  const double r1 = unit_decay_radius(unit, eps);
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = r1;
  return r1 * k.scale;
}

// ------------------------------------------------------------------ ES window and its transform
// phi(t) = exp(beta (sqrt(1-t^2) - 1)) - exp(-beta), |t| <= 1, t = (v - l)/(w/2)   (window choice: reading R6)
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& wts) {
  x.resize(n);
  wts.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      const double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-15) break;
    }
    x[i] = z;
    wts[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// Phi(xi) = int phi_win(v) e^{-2 pi i xi v} dv,  phi_win(v) = phi(v/(w/2))
static double es_exact(double t, double beta);

static double window_ft(double xi, int w, double beta, const std::vector<double>& gx, const std::vector<double>& gw) {
  const double half = 0.5 * w;
  double s = 0.0;
  for (size_t i = 0; i < gx.size(); ++i) {
    const double t = gx[i];
    s += gw[i] * es_exact(t, beta) * std::cos(2.0 * kPi * xi * half * t);
  }
  return half * s;
}

// ------------------------------------------------------------------ window polynomials (R6)
// ES window with its edge value subtracted, so that it vanishes continuously at |t| = 1 (better polynomial fits)
static double es_exact(double t, double beta) {
  if (std::fabs(t) >= 1.0) return 0.0;
  return std::exp(beta * (std::sqrt(1.0 - t * t) - 1.0)) - std::exp(-beta);
}

bool fit_window_poly(int w, double beta, float* coef, double* max_err) {
  const int D = kPolyDeg, n = D + 1;
  double worst = 0.0;
  for (int j = 0; j < w; ++j) {
    // interpolate at Chebyshev nodes of [0,1] (near-minimax), Vandermonde solve in fp64
    double A[n][n + 1];
    for (int i = 0; i < n; ++i) {
      const double f = 0.5 - 0.5 * std::cos(kPi * (i + 0.5) / n);
      double pw = 1.0;
      for (int k = 0; k < n; ++k) { A[i][k] = pw; pw *= f; }
      A[i][n] = es_exact((f + 0.5 * w - 1.0 - j) * 2.0 / w, beta);
    }
    for (int c = 0; c < n; ++c) {   // Gaussian elimination with partial pivoting
      int piv = c;
      for (int r = c + 1; r < n; ++r)
        if (std::fabs(A[r][c]) > std::fabs(A[piv][c])) piv = r;
      for (int k = 0; k <= n; ++k) std::swap(A[c][k], A[piv][k]);
      for (int r = 0; r < n; ++r) {
        if (r == c) continue;
        const double m = A[r][c] / A[c][c];
        for (int k = c; k <= n; ++k) A[r][k] -= m * A[c][k];
      }
    }
    for (int k = 0; k < n; ++k) coef[j * n + k] = static_cast<float>(A[k][n] / A[k][k]);
    for (int i = 0; i <= 400; ++i) {   // check the fp32 coefficients on a dense grid
      const double f = std::min(i / 400.0, 1.0 - 1e-12);
      double acc = 0.0;
      for (int k = D; k >= 0; --k) acc = acc * f + coef[j * n + k];
      worst = std::max(worst, std::fabs(acc - es_exact((f + 0.5 * w - 1.0 - j) * 2.0 / w, beta)));
    }
  }
  *max_err = worst;
  return worst < 1e-4;
}

// ------------------------------------------------------------------ data-independent window tables (R6)
// ES shape for the requested oversampling (Barnett et al. 2019 choice beta = 0.97 pi (1 - 1/(2 os)) w, os capped at
// 8); a slice's actual grid oversampling n_p / (2 (k_hi + 1)) is >= os (n_p is a power of two), where this window
// is only more accurate.  Phi is tabulated on j / n_cap (j <= n_cap / 2): the planner reads Phi(k / n_p) at
// j = k n_cap / n_p.  Cached per (w, os, n_cap).
const WindowTables& window_tables(int w, int os, int ncap) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, WindowTables> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(w, os, ncap);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  WindowTables t;
  t.w = w;
  t.beta = static_cast<float>(0.97 * kPi * (1.0 - 1.0 / (2.0 * std::min(os, 8))) * w);
  t.poly.assign(static_cast<size_t>(w) * (kPolyDeg + 1), 0.f);
  fit_window_poly(w, t.beta, t.poly.data(), &t.poly_err);
  std::vector<double> gx, gw;
  gauss_legendre(128, gx, gw);
  t.phi2inv.assign(ncap / 2 + 1, 0.f);
  for (int j = 0; j <= ncap / 2; ++j) {
    const double ph = window_ft(static_cast<double>(j) / ncap, w, t.beta, gx, gw);
    t.phi2inv[j] = static_cast<float>(1.0 / (ph * ph));
  }
  return cache.emplace(key, std::move(t)).first->second;
}

}  // namespace sks
