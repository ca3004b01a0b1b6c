/*
 * oracle.c -- CPU fp64 ORACLE for sliced fast kernel summation (arXiv 2401.08260).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2401_08260_b200/, libsks.so) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX source), DESIGN.md R# = a
 * reading of a passage where the paper is silent/ambiguous (listed in DESIGN.md).
 *
 * What it computes (plain definitions, fp64, no blocking / fusion / reordering):
 *   (a) or_exact_sum   s_m = sum_n w_n F(||x_n - y_m||)
 *   (b) or_sliced_sum  s_m = (1/P) sum_p sum_n w_n f(|<xi_p,x_n> - <xi_p,y_m>|) P:454, Alg.1
 *       with the 1D sums done directly (definition) instead of a fast engine.
 *   f = the 1D counterpart of F from Table 1 / Appendix C,
 *   evaluated from its defining power series (Thm 2.2); at d = 3 from the closed form
 *   f(t) = F(t) + t F'(t) of Cor 2.4, which needs no series.
 *   directions: DESIGN.md R1 (the paper only says "Draw P random directions").
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): brute force on tiny inputs with hand values,
 * d=1 (f=F) and d=3 (Cor 2.4) closed forms, the S_d quadrature of Prop 2.3
 * (P:161-163), Monte-Carlo slicing identities, E|<xi,z>| = ||z||/c_d,
 * 1F2 identities, SplitMix64 published test vector, slicing error ~ P^{-1/2} (Prop 2.6).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_GAUSSIAN = 0, OR_NEGDIST = 1, OR_LAPLACIAN = 2, OR_MATERN = 3 };

/* last error flag: set when a series evaluation is too ill-conditioned to trust */
static volatile int or_err_flag = 0;
int or_error(void) { return or_err_flag; }
void or_clear_error(void) { or_err_flag = 0; }

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------- constants */

/* c_d = sqrt(pi) Gamma((d+1)/2) / Gamma(d/2): Table 1 negative-distance row */
double or_cd(int d) {
  return sqrt(M_PI) * exp(lgamma(0.5 * (d + 1)) - lgamma(0.5 * d));
}

/* ------------------------------------------------------ hypergeometric series */

/* 1F1(a;b;z) = sum_n (a)_n/(b)_n z^n/n!  (the series named in Table 1).
 * Returns the sum; *maxterm receives max_n |term_n| (conditioning of the plain sum). */
static double hyp1f1_series(double a, double b, double z, double* maxterm) {
  double term = 1.0, sum = 1.0, mt = 1.0;
  for (int n = 0; n < 100000; ++n) {
    term *= (a + n) / (b + n) * z / (n + 1);
    sum += term;
    double at = fabs(term);
    if (at > mt) mt = at;
    if (term == 0.0) break;
    if (at < 1e-17 * fabs(sum) && n > fabs(z) + fabs(a)) break;
  }
  *maxterm = mt;
  return sum;
}

/* 1F2(a;b,c;z) = sum_n Gamma(n+a)/Gamma(a) Gamma(b)/Gamma(n+b) Gamma(c)/Gamma(n+c) z^n/n! */
static double hyp1f2_series(double a, double b, double c, double z, double* maxterm) {
  double term = 1.0, sum = 1.0, mt = 1.0;
  for (int n = 0; n < 100000; ++n) {
    term *= (a + n) / ((b + n) * (c + n)) * z / (n + 1);
    sum += term;
    double at = fabs(term);
    if (at > mt) mt = at;
    if (term == 0.0) break;
    if (at < 1e-17 * fabs(sum) && n > sqrt(fabs(z)) + fabs(a)) break;
  }
  *maxterm = mt;
  return sum;
}

double or_hyp1f1(double a, double b, double z) { double m; return hyp1f1_series(a, b, z, &m); }
double or_hyp1f2(double a, double b, double c, double z) { double m; return hyp1f2_series(a, b, c, z, &m); }

/* absolute error we accept from cancellation in a plain fp64 series */
#define OR_MAX_ABS_CANCEL 1e-9

/* ------------------------------------------------ radial basis functions F (d-dim) */

/* Matern nu = p + 1/2 closed form */
static double matern_halfint_F(int p, double beta, double x) {
  double q = sqrt(2.0 * p + 1.0) * x / beta;
  double fact_p = tgamma(p + 1.0), fact_2p = tgamma(2.0 * p + 1.0);
  double s = 0.0;
  for (int n = 0; n <= p; ++n)
    s += tgamma(p + n + 1.0) / (tgamma(n + 1.0) * tgamma(p - n + 1.0)) * pow(2.0 * q, p - n);
  return exp(-q) * fact_p / fact_2p * s;
}

/* F(r) for K(x,y)=F(||x-y||): Table 1, Laplacian exp(-alpha r) with alpha = 1/scale
 * (R8), Matern P:1163. param = sigma | (unused) | ell | beta. */
double or_F(int kind, double param, int mp, double r) {
  switch (kind) {
    case OR_GAUSSIAN: return exp(-r * r / (2.0 * param * param));
    case OR_NEGDIST: return -r;
    case OR_LAPLACIAN: return exp(-r / param);
    case OR_MATERN: return matern_halfint_F(mp, param, r);
  }
  return NAN;
}

/* ------------------------------------------------ 1D counterparts f (Table 1 / App. C) */

/* Gaussian: f(r) = 1F1(d/2; 1/2; -r^2/(2 sigma^2))  (Table 1, Lemma 2.5).
 * The plain series alternates; when it loses too many digits we use Kummer's transformation
 * 1F1(a;b;-x) = e^{-x} 1F1(b-a;b;x) (a textbook identity of the same function, terminating
 * for odd d).  If both forms are too ill-conditioned the oracle refuses (error flag). */
double or_f_gauss(double r, double sigma, int d) {
  double x = r * r / (2.0 * sigma * sigma);
  double a = 0.5 * d, b = 0.5;
  double m1, m2;
  double v1 = hyp1f1_series(a, b, -x, &m1);
  double e1 = m1 * 2.2e-16 * 8.0;
  if (e1 < 1e-13) return v1;
  double v2 = exp(-x) * hyp1f1_series(b - a, b, x, &m2);
  double e2 = exp(-x) * m2 * 2.2e-16 * 8.0;
  if (e2 < e1) { if (e2 > OR_MAX_ABS_CANCEL) or_err_flag = 1; return v2; }
  if (e1 > OR_MAX_ABS_CANCEL) or_err_flag = 1;
  return v1;
}

/* Laplacian F = exp(-alpha r): f(r) = 1F2(d/2;1/2,1/2;a^2r^2/4)
 *   - sqrt(pi) alpha r Gamma((d+1)/2)/Gamma(d/2) * 1F2((d+1)/2;1,3/2;a^2r^2/4) */
double or_f_laplace(double r, double alpha, int d) {
  double z = alpha * alpha * r * r / 4.0;
  double m1, m2;
  double s1 = hyp1f2_series(0.5 * d, 0.5, 0.5, z, &m1);
  double coef = alpha * r * or_cd(d);
  double s2 = hyp1f2_series(0.5 * (d + 1), 1.0, 1.5, z, &m2);
  double err = (m1 + coef * m2) * 2.2e-16 * 8.0;
  if (err > OR_MAX_ABS_CANCEL) or_err_flag = 1;
  return s1 - coef * s2;
}

/* Matern nu = p+1/2, length beta:
 * f(x) = 1F2(d/2;1/2,1-nu; nu x^2/(2b^2))
 *      - Gamma(1-nu)Gamma(nu+d/2) x^{2nu} (2nu)^nu / (Gamma(d/2)Gamma(2nu+1) b^{2nu})
 *        * 1F2(nu+d/2; nu+1/2, nu+1; nu x^2/(2b^2)) */
double or_f_matern(double r, double beta, int p, int d) {
  double nu = p + 0.5;
  double z = nu * r * r / (2.0 * beta * beta);
  double m1, m2;
  double s1 = hyp1f2_series(0.5 * d, 0.5, 1.0 - nu, z, &m1);
  /* Gamma(1-nu) is finite and may be negative for half-integer nu: use tgamma (sign kept) */
  double coef = tgamma(1.0 - nu) * exp(lgamma(nu + 0.5 * d) - lgamma(0.5 * d) - lgamma(2.0 * nu + 1.0)) *
                pow(r, 2.0 * nu) * pow(2.0 * nu, nu) / pow(beta, 2.0 * nu);
  double s2 = hyp1f2_series(nu + 0.5 * d, nu + 0.5, nu + 1.0, z, &m2);
  double err = (m1 + fabs(coef) * m2) * 2.2e-16 * 8.0;
  if (err > OR_MAX_ABS_CANCEL) or_err_flag = 1;
  return s1 - coef * s2;
}

/* negative distance: f(r) = -c_d r  (Table 1) */
double or_f_negdist(double r, int d) { return -or_cd(d) * r; }

/* d = 3: Cor 2.4 gives the counterpart in closed form, f(t) = F(t) + t F'(t), for any
 * differentiable F.  Written out for the three smooth kernels (F from Table 1 P:200-204 / P:1163):
 *   Gaussian  F = exp(-t^2/(2 s^2)):      t F' = -(t^2/s^2) F
 *   Laplacian F = exp(-t/ell):            t F' = -(t/ell) F
 *   Matern    F = C e^{-q} S(q), q = sqrt(2p+1) t/beta, S(q) = sum_n a_n (2q)^{p-n}:
 *             t F' = q dF/dq = C e^{-q} q (S'(q) - S(q)),  S'(q) = sum_{n<p} a_n 2 (p-n) (2q)^{p-n-1}.
 * These are exact (no series), so the oracle stays conditioned at any t for d = 3. */
static double f_d3(int kind, double param, int mp, double t) {
  switch (kind) {
    case OR_GAUSSIAN: {
      double u = t * t / (param * param);
      return (1.0 - u) * exp(-0.5 * u);
    }
    case OR_LAPLACIAN: {
      double u = t / param;
      return (1.0 - u) * exp(-u);
    }
    case OR_MATERN: {
      int p = mp;
      double q = sqrt(2.0 * p + 1.0) * t / param;
      double C = tgamma(p + 1.0) / tgamma(2.0 * p + 1.0);
      double S = 0.0, dS = 0.0;
      for (int n = 0; n <= p; ++n) {
        double a = tgamma(p + n + 1.0) / (tgamma(n + 1.0) * tgamma(p - n + 1.0));
        S += a * pow(2.0 * q, p - n);
        if (p - n >= 1) dS += a * 2.0 * (p - n) * pow(2.0 * q, p - n - 1);
      }
      return C * exp(-q) * (S + q * (dS - S));
    }
  }
  return NAN;
}

/* f by its defining series (Table 1 / App. C) at any d, bypassing the d = 3 closed form; used by the
 * pins that compare the two where the series is well conditioned. */
double or_f_series(int kind, double param, int mp, int d, double r) {
  switch (kind) {
    case OR_GAUSSIAN: return or_f_gauss(r, param, d);
    case OR_NEGDIST: return or_f_negdist(r, d);
    case OR_LAPLACIAN: return or_f_laplace(r, 1.0 / param, d);
    case OR_MATERN: return or_f_matern(r, param, mp, d);
  }
  return NAN;
}

double or_f(int kind, double param, int mp, int d, double r) {
  if (d == 3 && kind != OR_NEGDIST) return f_d3(kind, param, mp, r);
  switch (kind) {
    case OR_GAUSSIAN: return or_f_gauss(r, param, d);
    case OR_NEGDIST: return or_f_negdist(r, d);
    case OR_LAPLACIAN: return or_f_laplace(r, 1.0 / param, d);
    case OR_MATERN: return or_f_matern(r, param, mp, d);
  }
  return NAN;
}

void or_f_vec(int kind, double param, int mp, int d, const double* r, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_f(kind, param, mp, d, r[i]);
}
void or_f_series_vec(int kind, double param, int mp, int d, const double* r, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_f_series(kind, param, mp, d, r[i]);
}
void or_F_vec(int kind, double param, int mp, const double* r, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_F(kind, param, mp, r[i]);
}

/* ------------------------------------------------ directions (R1) */
/* SplitMix64 (Steele, Lea, Flood 2014) -- independent implementation of the spec in DESIGN.md */
uint64_t or_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* round a double to the nearest bf16 value (ties to even), returned as double.
 * Done as double -> float (RN) -> bf16 (RNE on the 16 dropped bits); exactness of the final
 * bf16 value is what matters: it is a float with 8 significand bits. */
double or_round_bf16(double v) {
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (double)f; /* inf/nan: not produced here */
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* g_p (unnormalised, bf16-exact) and 1/||g_p|| in fp64, for p in [p0,p1). xi_p = g_p * inv_norm_p. */
void or_directions(int P, int d, uint64_t seed, int p0, int p1, double* g, double* inv_norm) {
  (void)P;
  for (int p = p0; p < p1; ++p) {
    uint64_t key = or_splitmix64(seed ^ or_splitmix64((uint64_t)p));
    double* gp = g + (int64_t)(p - p0) * d;
    for (int q = 0; 2 * q < d; ++q) {
      uint64_t a = or_splitmix64(key + 2ULL * q);
      uint64_t b = or_splitmix64(key + 2ULL * q + 1ULL);
      double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53;
      double u2 = (double)(b >> 11) * 0x1.0p-53;
      double rad = sqrt(-2.0 * log(u1));
      double ang = 2.0 * M_PI * u2;
      gp[2 * q] = or_round_bf16(rad * cos(ang));
      if (2 * q + 1 < d) gp[2 * q + 1] = or_round_bf16(rad * sin(ang));
    }
    double ss = 0.0;
    for (int j = 0; j < d; ++j) ss += gp[j] * gp[j];
    inv_norm[p - p0] = 1.0 / sqrt(ss);
  }
}

/* ------------------------------------------------ projections P_xi(x) = <xi, x> */
/* z[p][i] = sum_j xi[p][j] * pts[i][j]; pts fp32 row-major (promoted exactly), xi fp64 */
void or_project(const float* pts, int64_t n, int d, const double* xi, int np, double* z) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int p = 0; p < np; ++p) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += xi[(int64_t)p * d + j] * (double)pts[i * d + j];
      z[(int64_t)p * n + i] = s;
    }
}

/* ------------------------------------------------ (a) exact d-dimensional sum */
void or_exact_sum(int kind, double param, int mp, int d, const float* x, int64_t N, const float* y,
                  const int64_t* tgt, int64_t n_tgt, const float* w, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_tgt; ++t) {
    const float* ym = y + tgt[t] * d;
    double s = 0.0;
    for (int64_t n = 0; n < N; ++n) {
      const float* xn = x + n * d;
      double r2 = 0.0;
      for (int j = 0; j < d; ++j) {
        double dd = (double)xn[j] - (double)ym[j];
        r2 += dd * dd;
      }
      s += (double)w[n] * or_F(kind, param, mp, sqrt(r2));
    }
    out[t] = s;
  }
}

/* ------------------------------------------------ (b) sliced estimator, direct 1D sums */
/* s_m = (1/P) sum_{p in [p0,p1)} sum_n w_n f(|<xi_p,x_n> - <xi_p,y_m>|)   (Alg.1 P:473-483,
 * 1D sums by definition).  xi: (p1-p0) x d fp64 unit vectors.  The 1/P uses the full P. */
void or_sliced_sum(int kind, double param, int mp, int d, const float* x, int64_t N, const float* y,
                   const int64_t* tgt, int64_t n_tgt, const float* w, int P, int p0, int p1,
                   const double* xi, double* out) {
  double* zx = (double*)malloc(sizeof(double) * (size_t)N);
  double* zy = (double*)malloc(sizeof(double) * (size_t)(n_tgt > 0 ? n_tgt : 1));
  for (int64_t t = 0; t < n_tgt; ++t) out[t] = 0.0;
  for (int p = p0; p < p1; ++p) {
    const double* xp = xi + (int64_t)(p - p0) * d;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += xp[j] * (double)x[n * d + j];
      zx[n] = s;
    }
    for (int64_t t = 0; t < n_tgt; ++t) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += xp[j] * (double)y[tgt[t] * d + j];
      zy[t] = s;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tgt; ++t) {
      double s = 0.0;
      for (int64_t n = 0; n < N; ++n) s += (double)w[n] * or_f(kind, param, mp, d, fabs(zx[n] - zy[t]));
      out[t] += s;
    }
  }
  for (int64_t t = 0; t < n_tgt; ++t) out[t] /= (double)P;
  free(zx);
  free(zy);
}

/* 1D sums on given projections (definition): t_m = sum_n w_n f(|zx_n - zy_m|) */
void or_sum_1d(int kind, double param, int mp, int d, const double* zx, const double* w, int64_t N,
               const double* zy, int64_t M, double* t) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t m = 0; m < M; ++m) {
    double s = 0.0;
    for (int64_t n = 0; n < N; ++n) s += w[n] * or_f(kind, param, mp, d, fabs(zx[n] - zy[m]));
    t[m] = s;
  }
}
