// plan.cu -- row a2 (the torus plan) on the device: one CTA per slice turns the slice's projection ranges (from
// the projection epilogue, or k_minmax for given projections) into its Fourier plan, with no host round trip.
//
// Per slice p (readings R3-R7b):
//   R_p = max - min of the slice's projections (x and y);  1/tau_p = R_p + r_eps (every aliased copy of the
//         counterpart lies beyond its eps decay radius, R3; Laplacian: also tau_p R_p <= 1/2 for the companion
//         h(u) = |u| - u^2 of R7);  cen_p = mid-range, u = tau_p (z - cen_p)                       (R4)
//   band [k_lo, k_hi]: the smallest band whose dropped coefficient mass (both signs of k) is <= eps / 2 at
//         each end, scanning |c_k| up to where the spectrum has decayed (R5; the same rule as the host's
//         sks_fourier_coeffs-based selection, evaluated by one warp with shuffle scans)
//   n_p = max(16, 2^ceil(log2(2 os (k_hi + 1))))  <= n_cap (else the call reports SKS_ERR_UNSUPPORTED)
//   D_p[k] = c_k(tau_p) / Phi(k / n_p)^2 on the band, 0 elsewhere: the diagonal with both NFFT deconvolutions
//         folded in (Phi = the window's transform, tabulated once on j / n_cap)
//   footprints: first cell / width of the x points' window support (spread) and of all points' (interpolation
//         polynomials), by the same fp32 operations as the spread / interpolation kernels
// and zeroes the slice's grid.  Every slice is planned from its own data only, so results do not depend on the
// slice batch or the number of GPUs.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace sks {

namespace {

constexpr int PL_T = 256;

__device__ __forceinline__ float key2f_pl(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// |c_k| of the periodised counterpart on period 1/tau (Lemma 2.5 P:304-306 for the Gaussian; R7 / R7b closed
// forms for the Laplacian's smooth part and the Matern): the same expressions as host.cpp torus_coeff
__device__ double torus_coeff_pl(const CoeffConst& c, double tau, int k) {
  const double PI = 3.14159265358979323846;
  const double rho = c.scale * tau * static_cast<double>(k);
  double fh = 0.0;
  if (c.kind == 0) {
    if (rho == 0.0) fh = (c.d == 1) ? sqrt(2.0 * PI) : 0.0;
    else {
      const double a = 2.0 * PI * PI * rho * rho;
      fh = exp(c.logpref - a + 0.5 * (c.d - 1) * log(a));
    }
  } else if (c.kind == 2) {
    const double s = 2.0 * PI * rho;
    if (s == 0.0) fh = (c.d == 1) ? 2.0 : 0.0;
    else fh = exp(c.logpref + (c.d - 1) * log(s) - 0.5 * (c.d + 1) * log1p(s * s));
  } else if (c.kind == 3) {
    const double lr = (c.d == 1) ? 0.0 : ((rho == 0.0) ? -INFINITY : (c.d - 1) * log(rho));
    fh = exp(c.logpref + lr - (c.nu + 0.5 * c.d) * log(2.0 * c.nu + 4.0 * PI * PI * rho * rho));
  }
  double v = tau * c.scale * fh;
  if (c.kind == 2) {
    const double A = c.lap_A / tau;
    v += (k == 0) ? A / 6.0 : -A / (2.0 * PI * PI * static_cast<double>(k) * static_cast<double>(k));
  }
  return v;
}

__device__ __forceinline__ double warp_incl_sum(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(PL_T) k_plan(const unsigned* __restrict__ mm, PlanConst pc,
                                               const float* __restrict__ phi2inv_cap, FPar* __restrict__ fp,
                                               float* __restrict__ D, float* __restrict__ grid,
                                               unsigned* __restrict__ flag16, unsigned* __restrict__ summary) {
  extern __shared__ double cabs[];   // |c_k|, k = 0 .. ncap / 2
  __shared__ int sK, sLo, sHi;
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int ncap = 1 << pc.ncap_log, KC = ncap / 2;
  if (flag16[0]) return;   // non-finite projections: the call fails, nothing to plan
  const float xmn = key2f_pl(mm[4 * p + 0]), xmx = key2f_pl(mm[4 * p + 1]);
  const float amn = key2f_pl(mm[4 * p + 2]), amx = key2f_pl(mm[4 * p + 3]);
  if (!(isfinite(xmn) && isfinite(xmx) && isfinite(amn) && isfinite(amx))) {
    if (tid == 0) atomicOr(flag16, 1u);
    return;
  }
  // torus scaling (R3, R7)
  const double R = static_cast<double>(amx) - static_cast<double>(amn);
  double inv_tau = R + pc.reps;
  if (pc.cc.kind == 2) inv_tau = fmax(inv_tau, 2.0 * R * (1.0 + 1e-6) + 1e-30);
  const float tauf = static_cast<float>(1.0 / inv_tau);
  const double tau = static_cast<double>(tauf);
  const float cen = static_cast<float>(0.5 * (static_cast<double>(amn) + static_cast<double>(amx)));
  const double half_eps = 0.5 * pc.eps;
  const bool gauss = pc.cc.kind == 0;

  // band (R5): |c_k| in chunks of PL_T until the spectrum has decayed (host rule: past the peak by 8, k > 16,
  // |c_k| < 1e-3 eps and the tail estimate < eps / 4; algebraic tails k^-4 sum to ~|c_k| k / 3)
  if (tid == 0) sK = -1;
  double peak = -1.0;
  int kpk = 0;
  // (a first chunk of 64: the narrow Gaussian bands stop inside it at a quarter of the fp64 transcendentals)
  for (int base = 0, chunk = 64; base <= KC; base += chunk, chunk = PL_T) {
    const int k = base + tid;
    if (tid < chunk && k <= KC) cabs[k] = fabs(torus_coeff_pl(pc.cc, tau, k));
    __syncthreads();
    if (tid < 32) {   // warp 0: running peak and the first k meeting the stop rule, 32 at a time
      for (int s0 = base; s0 < base + chunk && s0 <= KC && sK < 0; s0 += 32) {
        const int kk = s0 + lane;
        const double v = kk <= KC ? cabs[kk] : -1.0;
        // inclusive prefix argmax (first occurrence of the max, strict '>' as in a sequential scan)
        double pv = v;
        int pk = kk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double tv = __shfl_up_sync(0xffffffffu, pv, o);
          const int tk = __shfl_up_sync(0xffffffffu, pk, o);
          if (lane >= o && tv >= pv) { pv = tv; pk = tk; }
        }
        int kp = kpk;
        if (pv > peak) kp = pk;   // this prefix beats the running peak
        const double tail = gauss ? v : v * kk / 3.0;
        const bool stop = kk <= KC && kk > kp + 8 && kk > 16 && v < 1e-3 * pc.eps && tail < 0.25 * pc.eps;
        const unsigned b = __ballot_sync(0xffffffffu, stop);
        if (b) {
          if (lane == 0) sK = s0 + __ffs(b) - 1;
        } else {
          const double wv = __shfl_sync(0xffffffffu, pv, 31);
          const int wk = __shfl_sync(0xffffffffu, pk, 31);
          if (wv > peak) { peak = wv; kpk = wk; }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (sK >= 0) break;
  }
  if (sK < 0) {   // the spectrum has not decayed within n_cap / 2: the kernel is too narrow for the data's range
    if (tid == 0) atomicOr(flag16 + 2, 1u);
    return;
  }
  if (tid < 32) {
    const int K = sK;
    // upper edge: drop from the top while the dropped mass (x2 for +-k, + the analytic far tail) stays <= eps/2
    double dropped = gauss ? 0.0 : 2.0 * cabs[K] * K / 3.0;
    int hi = K;
    while (hi > 0) {
      const int kk = hi - lane;   // descending
      const double c2 = kk >= 1 ? 2.0 * cabs[kk] : 1e300;   // k = 0 is never dropped
      const double cum = dropped + warp_incl_sum(c2, lane);
      const unsigned ok = __ballot_sync(0xffffffffu, cum <= half_eps);
      const int cnt = __popc(~ok) == 0 ? 32 : __ffs(~ok) - 1;   // leading lanes that fit
      hi -= cnt;
      if (cnt < 32) break;
      dropped = __shfl_sync(0xffffffffu, cum, 31);
    }
    if (hi < 0) hi = 0;
    // lower edge (Gaussian bands sit on a bump away from 0 for d > 1): drop from the bottom
    int lo = 0;
    if (gauss) {
      double dl = 0.0;
      while (lo < hi) {
        const int kk = lo + lane;
        const double c = kk < hi ? (kk == 0 ? 1.0 : 2.0) * cabs[kk] : 1e300;
        const double cum = dl + warp_incl_sum(c, lane);
        const unsigned ok = __ballot_sync(0xffffffffu, cum <= half_eps);
        const int cnt = __popc(~ok) == 0 ? 32 : __ffs(~ok) - 1;
        lo += cnt;
        if (cnt < 32) break;
        dl = __shfl_sync(0xffffffffu, cum, 31);
      }
    }
    if (lane == 0) { sLo = lo; sHi = hi; }
  }
  __syncthreads();
  const int klo = sLo, khi = sHi;
  int logn = 4;
  while ((1 << logn) < 2 * pc.os * (khi + 1)) ++logn;
  const int n = 1 << logn;
  if (logn > pc.ncap_log || (pc.ndft && khi - klo + 1 > 32)) {
    if (tid == 0) atomicOr(flag16 + 2, logn > pc.ncap_log ? 1u : 2u);
    return;
  }
  // footprints: the spread / interpolation kernels' fp32 operation sequence (grid_coord, then - w/2)
  const float nf = static_cast<float>(n), hw = 0.5f * pc.w;
  const float taun = __fmul_rn(tauf, nf);   // n = 2^k: exact
  auto cell = [&](float z) { return floorf(__fsub_rn(__fmul_rn(__fsub_rn(z, cen), taun), hw)); };
  const int l0 = static_cast<int>(cell(xmn)), l1 = static_cast<int>(cell(xmx)) + pc.w + 1;   // one cell of margin
  const int la0 = static_cast<int>(cell(amn)), la1 = static_cast<int>(cell(amx)) + 2;
  SKS_CHECK(l1 - l0 + 1 >= pc.w + 2 && la1 - la0 + 1 >= 3 && la1 - la0 + 1 <= ncap + 16 && khi <= KC && klo <= khi);
  // diagonal: D[k] = c_k / Phi(k/n)^2 on the band (the NDFT has no window to undo)
  const int nh = n / 2 + 1, shift = pc.ncap_log - logn;
  float* Dp = D + static_cast<int64_t>(p) * (ncap / 2 + 1);
  for (int k = tid; k < nh; k += PL_T) {
    float v = 0.f;
    if (k >= klo && k <= khi) {
      const double c = torus_coeff_pl(pc.cc, tau, k);
      v = static_cast<float>(pc.ndft ? c : c * static_cast<double>(phi2inv_cap[k << shift]));
    }
    Dp[k] = v;
  }
  float* gp = grid + static_cast<int64_t>(p) * ncap;
  for (int l = tid; l < n; l += PL_T) gp[l] = 0.f;
  if (tid == 0) {
    FPar f;
    f.tau = tauf;
    f.cen = cen;
    f.lmin = l0;
    f.klo = klo;
    f.khi = khi;
    f.lminA = la0;
    f.logn = logn;
    f.W = l1 - l0 + 1;
    f.WA = la1 - la0 + 1;
    fp[p] = f;
    // call summary for sks_last_plan: max n, max k_hi, min k_lo, max W, max band, tau range (positive floats
    // order as unsigned), max WA
    atomicMax(summary + 0, static_cast<unsigned>(n));
    atomicMax(summary + 1, static_cast<unsigned>(khi));
    atomicMin(summary + 2, static_cast<unsigned>(klo));
    atomicMax(summary + 3, static_cast<unsigned>(f.W));
    atomicMax(summary + 4, static_cast<unsigned>(khi - klo + 1));
    atomicMin(summary + 5, __float_as_uint(tauf));
    atomicMax(summary + 6, __float_as_uint(tauf));
    atomicMax(summary + 7, static_cast<unsigned>(f.WA));
  }
}

}  // namespace

cudaError_t launch_plan(const unsigned* mm, int np, const PlanConst& pc, const float* phi2inv_cap, FPar* fp, float* D,
                        float* grid, unsigned* flag16, unsigned* summary, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((1 << pc.ncap_log) / 2 + 1);
  set_smem_attr_once(reinterpret_cast<const void*>(k_plan), static_cast<int>(smem));
  k_plan<<<np, PL_T, smem, st>>>(mm, pc, phi2inv_cap, fp, D, grid, flag16, summary);
  return cudaGetLastError();
}

}  // namespace sks
