// host.h -- host-side (C++) pieces of libsks: directions (R1) and the torus planner
// (Sec. 3.1 P:485-551 with readings R3-R7b).  Shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sks {

// ---- directions (R1): one SplitMix64 substream per slice p, Box-Muller in fp64, bf16 RNE
void make_directions(int P, int d, uint64_t seed, int p0, int p1, float* g, double* inv_norm);

// ---- kernel model: f(x) = f1(x/scale), f1 the unit-scale 1D counterpart (Table 1)
struct KernelModel {
  int kind;      // sks_kind
  int matern_p;  // nu = p + 1/2
  double scale;  // sigma | - | ell | beta
  int d;
};

double cd(int d);  // sqrt(pi) Gamma((d+1)/2)/Gamma(d/2)

// Fourier transform of the unit-scale counterpart: fhat1(rho) = int f1(x) e^{-2 pi i x rho} dx
//   Gaussian: Lemma 2.5 with sigma = 1; Laplacian / Matern: Fourier-slice identity (R7/R7b)
double fhat1(const KernelModel& k, double rho);

// torus coefficient c_k of the periodised counterpart on period 1/tau (R4, R7):
//   Gaussian / Matern: tau * fhat(tau k);  Laplacian smooth part: tau fhat(tau k) + (alpha c_d / tau) hhat_k
double torus_coeff(const KernelModel& k, double tau, int64_t kk);

// decay radius (in x units) beyond which |f(x)| <= eps  (reading R3): numeric Fourier integral, cached
double decay_radius(const KernelModel& k, double eps);

// Piecewise-polynomial form of the window (R6): for a point with fractional offset f in [0,1), tap j of w
// has weight p_j(f) = sum_k coef[j*(deg+1) + k] f^k ~= ES((f + w/2 - 1 - j) * 2/w).
// degree 7: the fit error is set by the ES window's edge kink, not by the degree (w = 6, os = 2: 6.7e-7 at
// degree 7 vs 5.1e-7 at 10), and 8 coefficients are two 16-byte loads per interpolation polynomial
constexpr int kPolyDeg = 7;
bool fit_window_poly(int w, double beta, float* coef /* w*(kPolyDeg+1) */, double* max_err);

// data-independent window data of the device planner (R6): ES shape, its piecewise-polynomial fit, and
// 1 / Phi(j / ncap)^2 for j = 0 .. ncap / 2 (window deconvolution, folded into D_k by the planner)
struct WindowTables {
  int w = 0;
  float beta = 0.f;
  std::vector<float> poly;      // w * (kPolyDeg + 1)
  double poly_err = 0.0;
  std::vector<float> phi2inv;   // [ncap / 2 + 1]
};
const WindowTables& window_tables(int w, int os, int ncap);

}  // namespace sks
