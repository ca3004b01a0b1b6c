// fused.cu -- rows a1 + a5 fused for the Fourier kernels at large N (the memory remark
// P:973-979): the projections of the SOURCES are spread into the slices' NFFT grids straight from the tensor-core
// accumulators, so they never reach HBM (cfg5 on one GPU: 20 GB of projection stores and as many loads saved).
//
//   k_sample_mean   mu = mean of a strided sample of the sources (fp64; any mu is valid, a central one is tight)
//   k_norm_bound    rho = max_n ||x_n - mu||, nmax = max_n ||x_n|| over all sources (one pass over X)
//   k_bound_ranges  per slice p: c_p = <xi_p, mu>; every source projection lies in [c_p - rho', c_p + rho']
//                   (Cauchy-Schwarz, ||xi_p|| = 1; rho' adds the projection's fp32 error bound), combined with
//                   the targets' exact ranges from their projection epilogue into the planner's ranges (R3: the
//                   torus must hold every point; a range bound instead of the exact x range only widens 1/tau)
//   k_proj_spread   persistent, one CTA per (slice tile of 128, range of 128-point source tiles):
//                   A = the tile's directions (resident in shared memory), B = the point tile (TMA, the raw fp32
//                   tile is the tf32 hi piece, converter warps form lo = rn_tf32(x - hi): TF32x2, reading R2),
//                   tcgen05.mma M = 128 slices x N = 128 points into double-buffered TMEM; epilogue warps own one
//                   slice each (TMEM lane = slice) and spread w_n phi(v - l) into the slice's private grid column
//                   in shared memory ([half][cell][slice]: conflict-free read-modify-writes, no atomics), flushed
//                   once per CTA with global atomics
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <cstring>

#include "kernels.h"
#include "tc_util.h"

namespace sks {

namespace {

using namespace tc;

// ------------------------------------------------------------------ range bound of the sources
constexpr int MEAN_ROWS = 2048, MEAN_PARTS = 32;   // sampled rows k N / MEAN_ROWS, summed in MEAN_PARTS groups

// part[g][j] = sum of dimension j over the sampled rows k = g, g + MEAN_PARTS, ... (fp64)
__global__ void __launch_bounds__(128) k_sample_mean_part(const float* __restrict__ x, int64_t N, int d,
                                                          double* __restrict__ part) {
  const int S = static_cast<int>(N < MEAN_ROWS ? N : MEAN_ROWS);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int k = blockIdx.x; k < S; k += MEAN_PARTS)   // (unrolled: the rows' loads in flight together, same order of adds)
      s += static_cast<double>(__ldg(x + (static_cast<int64_t>(k) * N / S) * d + j));
    part[static_cast<int64_t>(blockIdx.x) * d + j] = s;
  }
}

// mu[j] = (sum over the parts, in order) / S; also zeroes the norm-bound words nb[0..7]
__global__ void k_sample_mean_fin(int64_t N, int d, const double* __restrict__ part, double* __restrict__ mu,
                                  unsigned* __restrict__ nb) {
  const int S = static_cast<int>(N < MEAN_ROWS ? N : MEAN_ROWS);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < MEAN_PARTS; ++g) s += part[static_cast<int64_t>(g) * d + j];
    mu[j] = s / S;
  }
  if (threadIdx.x < 8) nb[threadIdx.x] = 0u;
}

// The fused kernels' operands (reading R2, FP16x2 with one scale per 8-row group): for the group's rows
//   s_g = 2^(14 - e), max |x| over the group = m 2^e (m in [0.5, 1)): s_g max|x| < 2^14 (s_g = 1 for a zero group)
//   hi = f16_rn(s_g x), lo = f16_rn(s_g x - hi)         (|s_g x - hi - lo| <= 2^-22 |s_g x| + 2^-25)
// stored as two fp16 arrays [rows][dp16] (dp16 = d rounded up to 8, pad columns zero) and rs[g] = 1 / (2^8 s_g):
// the tensor cores accumulate (2^8 g) . (s_g x) exactly in fp32 (directions fp16 x 2^8, exact: R1), and the
// epilogues' rs[g] (a power of two) restores <g, x> without rounding.
constexpr int PR_G = 8;    // rows per scale group: one warp holds a group in registers (one float4 per lane and row)

__device__ __forceinline__ float group_scale(float m) {   // s_g from the group's max |x| (finite, >= 0)
  if (!(m > 0.f) || !(m < 3.0e38f)) return 1.0f;
  int e;
  frexpf(m, &e);
  e = e < -100 ? -100 : e;
  return ldexpf(1.0f, 14 - e);
}

// one warp per 8-row group (grid-stride), lane l dims 4 l .. 4 l + 3 (d <= 128), one pass over the rows:
// out[0] = max ||x - mu||^2, out[1] = max ||x||^2 (float bits: non-negative floats order as unsigned ints),
// out[2] = non-finite seen; the group's fp16 hi / lo rows and rs[g]; with w, the weights zero padded (wpad)
__global__ void __launch_bounds__(256, 4) k_prep_f16(const float* __restrict__ x, int64_t N, int d, int dp16,
                                                  const double* __restrict__ mu, unsigned* __restrict__ out,
                                                  __half* __restrict__ xh, __half* __restrict__ xl,
                                                  float* __restrict__ rs, const float* __restrict__ w,
                                                  float* __restrict__ wpad) {
  __shared__ float smu[128];
  for (int j = threadIdx.x; j < 128; j += blockDim.x) smu[j] = j < d ? static_cast<float>(mu[j]) : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const bool on = 4 * lane < d, pad = 4 * lane < dp16;
  const float4 m4 = on ? make_float4(smu[4 * lane], smu[4 * lane + 1], smu[4 * lane + 2], smu[4 * lane + 3])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
  float r2max = 0.f, n2max = 0.f;
  bool bad = false;
  const int64_t ngroups = (N + 127) / 128 * (128 / PR_G);   // whole 128-row tiles (rs and wpad cover them)
  // the warp index as a visibly warp-uniform value (launched with 8 warps): the loop's shuffles then compile without
  // divergence handling (a threadIdx-derived bound made ptxas wrap each one, at 2.5x the registers)
  const int64_t w0 = blockIdx.x * 8 + __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int64_t nw = static_cast<int64_t>(gridDim.x) * 8;
  for (int64_t g = w0; g < ngroups; g += nw) {
    const int64_t r0 = g * PR_G;
    if (w && lane < PR_G) wpad[r0 + lane] = r0 + lane < N ? __ldg(w + r0 + lane) : 0.f;
    float4 v[PR_G];
#pragma unroll
    for (int u = 0; u < PR_G; ++u) {   // all loads in flight first (streamed once)
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (on && r0 + u < N) v[u] = __ldcs(reinterpret_cast<const float4*>(x + (r0 + u) * d) + lane);
    }
    float am = 0.f;
#pragma unroll
    for (int u = 0; u < PR_G; ++u) {
      am = fmaxf(am, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
      const float a = v[u].x - m4.x, b = v[u].y - m4.y, c = v[u].z - m4.z, e = v[u].w - m4.w;
      float r2 = fmaf(a, a, fmaf(b, b, fmaf(c, c, e * e)));
      float n2 = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, fmaf(v[u].z, v[u].z, v[u].w * v[u].w)));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      }
      bad |= !isfinite(n2);
      r2max = fmaxf(r2max, r2);
      n2max = fmaxf(n2max, n2);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
    const float sg = group_scale(am);
    if (lane == 0) rs[g] = 1.0f / (256.0f * sg);   // (exact: a power of two)
    // (no early continue: the shuffles above must stay convergent)
#pragma unroll
    for (int u = 0; u < PR_G; ++u) {
      const int64_t r = r0 + u;
      if (!pad || r >= N) continue;
      const float a0 = v[u].x * sg, a1 = v[u].y * sg, a2 = v[u].z * sg, a3 = v[u].w * sg;
      const __half2 h01 = __floats2half2_rn(a0, a1), h23 = __floats2half2_rn(a2, a3);
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      const __half2 l01 = __floats2half2_rn(a0 - f01.x, a1 - f01.y), l23 = __floats2half2_rn(a2 - f23.x, a3 - f23.y);
      uint2 hv, lv;
      hv.x = *reinterpret_cast<const uint32_t*>(&h01);
      hv.y = *reinterpret_cast<const uint32_t*>(&h23);
      lv.x = *reinterpret_cast<const uint32_t*>(&l01);
      lv.y = *reinterpret_cast<const uint32_t*>(&l23);
      __stcs(reinterpret_cast<uint2*>(xh + r * dp16) + lane, hv);
      __stcs(reinterpret_cast<uint2*>(xl + r * dp16) + lane, lv);
    }
  }
  if (lane == 0) {
    if (r2max > 0.f) atomicMax(out + 0, __float_as_uint(r2max));
    if (n2max > 0.f) atomicMax(out + 1, __float_as_uint(n2max));
    if (bad) atomicOr(out + 2, 1u);
  }
}

__device__ __forceinline__ unsigned f2key_fu(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f_fu(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// rho' = rho (1 + 2^-10) + 2^-19 nmax from the norm words {max ||z - mu||^2, max ||z||^2}: the fp32 sums of squares
// (relative error <= d 2^-24 <= 2^-17 for d <= 128, halved by the root) and the projection's error (<= 2^-21 ||z||,
// DESIGN.md R2) are far inside these margins
__device__ __forceinline__ double bound_radius(const unsigned* nb) {
  return sqrt(static_cast<double>(__uint_as_float(nb[0]))) * (1.0 + 0x1p-10) +
         sqrt(static_cast<double>(__uint_as_float(nb[1]))) * 0x1p-19;
}

// one warp per slice: c_p = <g_p, mu> inv_p (fp64); every projection of the bounded set lies in [c_p - rho',
// c_p + rho'] (Cauchy-Schwarz, ||xi_p|| = 1).  mm[p] = {xmin, xmax, allmin, allmax}: x from its bound (nb[0..2]);
// all = the hull of the x bound and either the targets' bound (ybound: nb[4..6]) or their exact range (their
// projection epilogue wrote it into mm[p][2..3])
__global__ void k_bound_ranges(const float* __restrict__ g32, int dp32, int d, const float* __restrict__ inv_norm,
                               int np, const double* __restrict__ mu, const unsigned* __restrict__ nb, int ybound,
                               unsigned* __restrict__ mm, unsigned* __restrict__ flag16) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= np) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s += static_cast<double>(g32[static_cast<int64_t>(p) * dp32 + j]) * mu[j];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane) return;
  if (nb[2] || (ybound && nb[6])) {
    atomicOr(flag16, 1u);
    return;
  }
  const double c = s * static_cast<double>(inv_norm[p]);
  const double rx = bound_radius(nb);
  const float xlo = nextafterf(static_cast<float>(c - rx), -CUDART_INF_F);
  const float xhi = nextafterf(static_cast<float>(c + rx), CUDART_INF_F);
  float ymn, ymx;
  if (ybound) {
    const double ry = bound_radius(nb + 4);
    ymn = nextafterf(static_cast<float>(c - ry), -CUDART_INF_F);
    ymx = nextafterf(static_cast<float>(c + ry), CUDART_INF_F);
  } else {
    ymn = key2f_fu(mm[4 * p + 2]);
    ymx = key2f_fu(mm[4 * p + 3]);
  }
  mm[4 * p + 0] = f2key_fu(xlo);
  mm[4 * p + 1] = f2key_fu(xhi);
  mm[4 * p + 2] = f2key_fu(fminf(xlo, ymn));
  mm[4 * p + 3] = f2key_fu(fmaxf(xhi, ymx));
}

// ------------------------------------------------------------------ the fused projection + spread
constexpr int FS_S = 128;          // slices per tile (UMMA M = TMEM lanes)
constexpr int FS_P = 128;          // points per tile (UMMA N)
constexpr int FS_STAGES = 2;       // (one tile of lookahead: the MMAs are far ahead of the epilogue)
constexpr int FS_KBMAX = 2;        // k-blocks of 64 fp16 dims (128-byte rows): d <= 128
constexpr int FS_WCAP = 32;        // private grid cells per slice (wider footprints: global atomics)
constexpr int FS_EPI = 16;         // epilogue warps: 4 per TMEM lane quadrant, 32 points of the tile each
constexpr int FS_NCOL = 2 * (FS_EPI / 4);   // private grid copies per slice: one per (point group, point parity)
// warp roles: w0 .. FS_EPI - 1 epilogue, then TMEM alloc, -, TMA producer, MMA issuer.  The issuers take the highest
// warp ids: the warp scheduler prefers the highest ready warp id, so the single-thread MMA loop is never starved
// of issue slots by the busy epilogue warps of its SM sub-partition
constexpr int FS_WALLOC = FS_EPI, FS_WTMA = FS_EPI + 2, FS_WMMA = FS_EPI + 3;
constexpr int FS_THREADS = 32 * (4 + FS_EPI);
constexpr int FS_PIECE = FS_P * 128;                      // one k-block of 128 points: 16 KB
constexpr int FS_A = FS_S * 128;                          // one k-block of the directions: 16 KB
constexpr int FS_OFF_STAGE = FS_KBMAX * FS_A;             // 32 KB of resident directions
constexpr int FS_OFF_GRID = FS_OFF_STAGE + FS_STAGES * 2 * FS_PIECE;
constexpr int FS_OFF_W = FS_OFF_GRID + FS_NCOL * FS_WCAP * FS_S * 4;   // the tiles' weights [2][FS_P]
constexpr int FS_OFF_BAR = FS_OFF_W + 2 * FS_P * 4;
constexpr int FS_SMEM = FS_OFF_BAR + 512 + 1024;          // + barriers, TMEM slot, window coefficients, alignment
static_assert(FS_SMEM <= 227 * 1024, "k_proj_spread shared memory");

// NC private copies of WCAP = 256 / NC cells per slice: 8 x 32 (a copy per point group and point parity), 4 x 64
// (a copy per point group), or one shared column of 256 cells updated with shared-memory atomics (fp32 atomicAdd on
// shared memory is a CAS loop on sm_100a, ~3x the cost of a private read-modify-write, against ~35x for the global
// atomics a slice beyond 256 cells falls back to).  The footprints are known on the device only (the planner's
// FPar.W), so all three variants are launched and each slice tile is taken by exactly one of them, by the widest
// footprint among its slices (<= 32, <= 64, wider); the other variants' CTAs of that tile exit at once
template <int WT, int NC>
__global__ void __launch_bounds__(FS_THREADS, 1)
    k_proj_spread(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXlo, int nk, int klast, int64_t N,
                  int np, int ranges, const float* __restrict__ rs, const float* __restrict__ inv_norm,
                  const float* __restrict__ wpad, const FPar* __restrict__ fp, PolyWin pw, int ncap,
                  float* __restrict__ grid,
                  const unsigned* __restrict__ flag16) {
  if (call_failed(flag16)) return;
  {
    const int ps = (blockIdx.x % ((np + FS_S - 1) / FS_S)) * FS_S + static_cast<int>(threadIdx.x);
    const int wps = (threadIdx.x < FS_S && ps < np) ? fp[ps].W : 0;
    const int b32 = __syncthreads_or(wps > FS_WCAP), b64 = __syncthreads_or(wps > 2 * FS_WCAP);
    const int cls = b64 ? 2 : (b32 ? 1 : 0);
    if (cls != (NC == FS_NCOL ? 0 : (NC == 1 ? 2 : 1))) return;   // (block-uniform) another variant's tile
  }
  extern __shared__ unsigned char fsraw[];
  // aligned by pointer arithmetic on the __shared__ array: the compiler keeps the shared state space (LDS / STS,
  // not generic LD / ST)
  unsigned char* sm = fsraw + ((1024u - (smem_u32(fsraw) & 1023u)) & 1023u);
  constexpr int WCAP = FS_NCOL * FS_WCAP / NC;   // private cells per slice and copy
  constexpr int WH = (WT + 1) / 2;               // mirror pairs (+ the middle tap of an odd window)
  static_assert(NC == FS_NCOL || NC == FS_EPI / 4 || NC == 1, "copies: per point group and parity, per group, one");
  float* priv = reinterpret_cast<float*>(sm + FS_OFF_GRID);   // [NC][WCAP][FS_S]
  uint64_t* afull = reinterpret_cast<uint64_t*>(sm + FS_OFF_BAR);
  uint64_t* xfull = afull + 1;                 // [FS_STAGES] raw tile (hi) and lo piece landed
  uint64_t* empty = xfull + FS_STAGES;         // [FS_STAGES] consumed by the MMAs
  uint64_t* tfull = empty + FS_STAGES;         // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint64_t* wfull = tempty + 2;                // [2] the tile's weights landed (slot b = the TMEM buffer's)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 2);
  const float* wsm = reinterpret_cast<const float*>(sm + FS_OFF_W);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int st_idx = blockIdx.x % ((np + FS_S - 1) / FS_S), r = blockIdx.x / ((np + FS_S - 1) / FS_S);
  const int64_t ntp = (N + FS_P - 1) / FS_P;
  const int64_t t0 = r * ntp / ranges, t1 = (r + 1) * ntp / ranges;   // this CTA's point tiles
  const int s0 = st_idx * FS_S;

  for (int e = threadIdx.x; e < FS_NCOL * FS_WCAP * FS_S; e += FS_THREADS) priv[e] = 0.f;
  if (warp == 0 && lane == 0) {
    mbar_init(afull, 1);
    for (int s = 0; s < FS_STAGES; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], FS_EPI);
      mbar_init(&wfull[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmXlo)) : "memory");
  }
  if (warp == FS_WALLOC) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * FS_P));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == FS_WTMA && lane == 0) {
    // ---- TMA producer: the tile's directions (fp16 x 2^8) once, then the point tiles' fp16 hi and lo pieces
    //      (written by the k_prep_f16 pass)
    mbar_expect_tx(afull, nk * FS_A);
    for (int kb = 0; kb < nk; ++kb) tma_load_2d(&tmA, afull, sm + kb * FS_A, kb * 64, s0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* sa = sm + FS_OFF_STAGE + stage * 2 * FS_PIECE;
        mbar_expect_tx(&xfull[stage], 2 * FS_PIECE);
        tma_load_2d(&tmX, &xfull[stage], sa, kb * 64, static_cast<int>(t * FS_P));
        tma_load_2d(&tmXlo, &xfull[stage], sa + FS_PIECE, kb * 64, static_cast<int>(t * FS_P));
        if (++stage == FS_STAGES) { stage = 0; phase ^= 1; }
      }
      // the tile's 128 weights (zero padded beyond N) into slot b, free once the epilogue of tile t - 2 released
      // TMEM buffer b
      const int b = it & 1;
      mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
      mbar_expect_tx(&wfull[b], FS_P * 4);
      bulk_load_1d(sm + FS_OFF_W + b * FS_P * 4, wpad + t * FS_P, FS_P * 4, &wfull[b]);
    }
  } else if (warp == FS_WMMA && lane == 0) {
    // ---- MMA issuer: D[slice][point] += A (2^8 g, fp16-exact) . B (s_t x: hi, then lo), K = 16 per MMA
    constexpr uint32_t idesc = idesc_f16(FS_S, FS_P);
    mbar_wait(afull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int b = it & 1;
      mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(b * FS_P);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&xfull[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned char* sb = sm + FS_OFF_STAGE + stage * 2 * FS_PIECE;
        const uint64_t da = umma_desc_sw128(sm + kb * FS_A);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint64_t db = umma_desc_sw128(sb + q * FS_PIECE);
#pragma unroll
          for (int k = 0; k < 4; ++k) {   // 4 MMAs of K = 8 tf32 (32 bytes) per 128-byte row
            if (kb == nk - 1 && k >= klast) break;   // (k-steps wholly in the zero padding beyond d)
            const uint32_t acc = (kb > 0 || q > 0 || k > 0) ? 1u : 0u;
            const uint64_t adv = static_cast<uint64_t>((k * 32) >> 4);
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                "l"(da + adv), "l"(db + adv), "r"(idesc), "r"(acc));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[stage]))
                     : "memory");
        if (++stage == FS_STAGES) { stage = 0; phase ^= 1; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&tfull[b]))
                   : "memory");
    }
  } else if (warp < FS_EPI) {
    // ---- epilogue: warp w owns TMEM lane quadrant q = w % 4 (slices s0 + 32 q + lane) and the 32 points
    //      h = (w - 8) / 4 of the tile; per point: the grid coordinate a = acc (tau_p n_p / ||g_p||) - (cen_p tau_p
    //      n_p + w/2) (one FMA; the planner's footprint has a cell of margin either side and the cell index is
    //      clamped to the private column), WT taps of the window polynomial (centred even / odd form), w_n-weighted
    //      into the slice's private column (cell-major: bank = lane, conflict-free)
    const int q = warp & 3, h = warp >> 2;
    const int p = s0 + 32 * q + lane;
    const bool live = p < np;
    FPar f{};
    float inv = 0.f;
    if (live) {
      f = fp[p];
      inv = inv_norm[p];
    }
    const int n = 1 << f.logn;
    const float taun = f.tau * static_cast<float>(n);
    const float ga = inv * taun, gb = -fmaf(f.cen, taun, 0.5f * pw.w);
    const int W = f.W;
    const bool wide = W > WCAP;   // (footprint beyond the private column: global atomics for this slice)
    // NC = 8: two private copies of the slice's column per warp, for the even and the odd points of a pair: the
    // pair's read-modify-writes cannot alias, so both points' loads are issued before either's stores.  NC = 4: one
    // copy per warp, the two points' read-modify-writes in order
    constexpr int CPW = NC / (FS_EPI / 4);                           // copies per warp (0: one copy for all warps)
    float* col = priv + (CPW * h * WCAP) * FS_S + 32 * q + lane;     // cell c at col[c * FS_S] (even points)
    float* colo = col + (CPW == 2 ? WCAP * FS_S : 0);                // (odd points)
    float* gp = grid + static_cast<int64_t>(live ? p : 0) * ncap;
    // window coefficients through shared memory into registers (read from the parameter bank, ptxas would
    // re-load them inside the loop)
    float* eos = reinterpret_cast<float*>(sm + FS_OFF_BAR + 256);   // [WH][8]
    if (threadIdx.x < WH * 8) eos[threadIdx.x] = pw.eo[threadIdx.x / 8][threadIdx.x % 8];   // (warps 0, 1: epilogue)
    asm volatile("bar.sync 1, %0;" ::"r"(FS_EPI * 32) : "memory");
    float E[WH][4], O[WH][4];
#pragma unroll
    for (int j = 0; j < WH; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        E[j][k] = eos[8 * j + k];
        O[j][k] = eos[8 * j + 4 + k];
      }
    const int cmax = W - WT;   // last admissible first-tap cell (relative to lmin)
    const bool fast = live && !wide;   // (dead lanes of the last slice tile and wide footprints: the slow loop)
    int it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int b = it & 1;
      const int c0 = h * 32;
      const int64_t i0 = t * FS_P + c0;
      const float* rsg = rs + 16 * t + 4 * h;   // the 8-point groups' 1 / (2^8 s_g) (powers of two: exact)
      mbar_wait_sleep(&tfull[b], (it >> 1) & 1);
      mbar_wait(&wfull[b], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem_base + static_cast<uint32_t>(b * FS_P + c0) + (static_cast<uint32_t>(32 * q) << 16);
      const float4* w4 = reinterpret_cast<const float4*>(wsm + b * FS_P + c0);
      const int nj = (N - i0 < 32) ? static_cast<int>(N - i0) : 32;
#pragma unroll 1
      for (int j0 = 0; j0 < 32; j0 += 8) {   // 8 columns (points) per TMEM load: few registers held
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr + j0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const float gat = ga * __ldg(rsg + j0 / 8);   // (the 8 points are one scale group)
        // the 8 points' weights: two 16-byte broadcast loads (every lane reads the same address; zero beyond N)
        const float4 wa = w4[j0 / 4], wb = w4[j0 / 4 + 1];
        const float w8[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
        if (fast) {
          // branch-free: points beyond N carry weight 0 (their rows are zero-filled by TMA; the clamp keeps their
          // cell in range).  Two points per step: the grid coordinate and the window polynomials of both in packed
          // fp32x2 FMAs (FFMA2, the same operations and rounding as the scalar form), then the two points'
          // read-modify-writes one after the other (their cells may coincide)
#pragma unroll
          for (int jj = 0; jj < 8; jj += 2) {
            const float2 a = __ffma2_rn(make_float2(__uint_as_float(v[jj]), __uint_as_float(v[jj + 1])),
                                        make_float2(gat, gat), make_float2(gb, gb));
            const float2 fl = make_float2(floorf(a.x), floorf(a.y));
            const float2 u = __fadd2_rn(__fadd2_rn(a, make_float2(-fl.x, -fl.y)), make_float2(-0.5f, -0.5f));
            const float2 u2 = __fmul2_rn(u, u);
            const int cl0 = min(max(static_cast<int>(fl.x) + 1 - f.lmin, 0), cmax);   // (memory safety only)
            const int cl1 = min(max(static_cast<int>(fl.y) + 1 - f.lmin, 0), cmax);
            SKS_CHECK(w8[jj] == 0.f || cl0 == static_cast<int>(fl.x) + 1 - f.lmin);   // the bound holds: no clamping
            SKS_CHECK(w8[jj + 1] == 0.f || cl1 == static_cast<int>(fl.y) + 1 - f.lmin);
            float2 tl[WH], th[WH];   // taps m and WT - 1 - m of both points (odd WT: tl[WT / 2] the middle tap)
#pragma unroll
            for (int m = 0; m < WH; ++m) {
              const float2 Em = __ffma2_rn(
                  __ffma2_rn(__ffma2_rn(make_float2(E[m][3], E[m][3]), u2, make_float2(E[m][2], E[m][2])), u2,
                             make_float2(E[m][1], E[m][1])),
                  u2, make_float2(E[m][0], E[m][0]));
              const float2 Om = __ffma2_rn(
                  __ffma2_rn(__ffma2_rn(make_float2(O[m][3], O[m][3]), u2, make_float2(O[m][2], O[m][2])), u2,
                             make_float2(O[m][1], O[m][1])),
                  u2, make_float2(O[m][0], O[m][0]));
              tl[m] = __ffma2_rn(u, Om, Em);
              th[m] = __ffma2_rn(make_float2(-u.x, -u.y), Om, Em);
            }
            float* c0p = col + cl0 * FS_S;    // even point: copy 0
            float* c1p = colo + cl1 * FS_S;   // odd point: copy 1
            float g0[WT], g1[WT];
            if constexpr (CPW == 2) {
#pragma unroll
              for (int m = 0; m < WT; ++m) {   // all 2 WT loads first (disjoint copies: no ordering needed)
                g0[m] = c0p[m * FS_S];
                g1[m] = c1p[m * FS_S];
              }
#pragma unroll
              for (int m = 0; m < WT / 2; ++m) {
                c0p[m * FS_S] = fmaf(w8[jj], tl[m].x, g0[m]);
                c0p[(WT - 1 - m) * FS_S] = fmaf(w8[jj], th[m].x, g0[WT - 1 - m]);
                c1p[m * FS_S] = fmaf(w8[jj + 1], tl[m].y, g1[m]);
                c1p[(WT - 1 - m) * FS_S] = fmaf(w8[jj + 1], th[m].y, g1[WT - 1 - m]);
              }
              if constexpr (WT & 1) {
                c0p[(WT / 2) * FS_S] = fmaf(w8[jj], tl[WT / 2].x, g0[WT / 2]);
                c1p[(WT / 2) * FS_S] = fmaf(w8[jj + 1], tl[WT / 2].y, g1[WT / 2]);
              }
            } else if constexpr (CPW == 0) {   // one column shared by the CTA's warps: shared-memory atomics
#pragma unroll
              for (int m = 0; m < WT / 2; ++m) {
                atomicAdd(c0p + m * FS_S, w8[jj] * tl[m].x);
                atomicAdd(c0p + (WT - 1 - m) * FS_S, w8[jj] * th[m].x);
                atomicAdd(c1p + m * FS_S, w8[jj + 1] * tl[m].y);
                atomicAdd(c1p + (WT - 1 - m) * FS_S, w8[jj + 1] * th[m].y);
              }
              if constexpr (WT & 1) {
                atomicAdd(c0p + (WT / 2) * FS_S, w8[jj] * tl[WT / 2].x);
                atomicAdd(c1p + (WT / 2) * FS_S, w8[jj + 1] * tl[WT / 2].y);
              }
            } else {   // one copy: the even point's stores before the odd point's loads (their cells may coincide)
#pragma unroll
              for (int m = 0; m < WT; ++m) g0[m] = c0p[m * FS_S];
#pragma unroll
              for (int m = 0; m < WT / 2; ++m) {
                c0p[m * FS_S] = fmaf(w8[jj], tl[m].x, g0[m]);
                c0p[(WT - 1 - m) * FS_S] = fmaf(w8[jj], th[m].x, g0[WT - 1 - m]);
              }
              if constexpr (WT & 1) c0p[(WT / 2) * FS_S] = fmaf(w8[jj], tl[WT / 2].x, g0[WT / 2]);
#pragma unroll
              for (int m = 0; m < WT; ++m) g1[m] = c1p[m * FS_S];
#pragma unroll
              for (int m = 0; m < WT / 2; ++m) {
                c1p[m * FS_S] = fmaf(w8[jj + 1], tl[m].y, g1[m]);
                c1p[(WT - 1 - m) * FS_S] = fmaf(w8[jj + 1], th[m].y, g1[WT - 1 - m]);
              }
              if constexpr (WT & 1) c1p[(WT / 2) * FS_S] = fmaf(w8[jj + 1], tl[WT / 2].y, g1[WT / 2]);
            }
          }
        } else if (live) {   // footprint wider than the private column: global atomics for this slice
          for (int jj = 0; jj < 8; ++jj) {
            const float wi = w8[jj];
            if (j0 + jj >= nj) continue;
            const float a = fmaf(__uint_as_float(v[jj]), gat, gb), fl = floorf(a);
            const float u = (a - fl) - 0.5f, u2 = u * u;
            const int cl = min(max(static_cast<int>(fl) + 1 - f.lmin, 0), cmax);
            for (int m = 0; m < WT / 2; ++m) {
              const float Em = fmaf(fmaf(fmaf(E[m][3], u2, E[m][2]), u2, E[m][1]), u2, E[m][0]);
              const float Om = fmaf(fmaf(fmaf(O[m][3], u2, O[m][2]), u2, O[m][1]), u2, O[m][0]);
              atomicAdd(&gp[(f.lmin + cl + m) & (n - 1)], wi * fmaf(u, Om, Em));
              atomicAdd(&gp[(f.lmin + cl + WT - 1 - m) & (n - 1)], wi * fmaf(-u, Om, Em));
            }
            if (WT & 1) {
              constexpr int m = WT / 2;
              const float Em = fmaf(fmaf(fmaf(E[m][3], u2, E[m][2]), u2, E[m][1]), u2, E[m][0]);
              const float Om = fmaf(fmaf(fmaf(O[m][3], u2, O[m][2]), u2, O[m][1]), u2, O[m][0]);
              atomicAdd(&gp[(f.lmin + cl + m) & (n - 1)], wi * fmaf(u, Om, Em));
            }
          }
        }
      }
      // the accumulator is read: release it to the MMAs of tile t + 2
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {   // flush: the NC private columns of each slice, one atomic per cell
    const int q = warp & 3, p = s0 + 32 * q + lane;
    if (p < np) {
      const FPar f = fp[p];
      const int n = 1 << f.logn;
      if (f.W <= WCAP) {
        float* gp = grid + static_cast<int64_t>(p) * ncap;
        const float* c0 = priv + 32 * q + lane;
        for (int c = 0; c < f.W; ++c) {
          float s = 0.f;
#pragma unroll
          for (int g = 0; g < NC; ++g) s += c0[(g * WCAP + c) * FS_S];
          if (s != 0.f) atomicAdd(&gp[(f.lmin + c) & (n - 1)], s);
        }
      }
    }
  }
  if (warp == FS_WALLOC) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * FS_P));
}

// ------------------------------------------------------------------ the fused projection + interpolation
// Rows a1 + a7 for the TARGETS: persistent, one CTA per (slice group of 128, range of 128-point target tiles);
// A = the target tile (TMA, FP16x2 as above), B = the group's directions (resident), tcgen05.mma M = 128 targets x
// N = 128 slices into double-buffered TMEM (TMEM lane = target).  The group's interpolation polynomials Q (written by
// k_fft_filter, economised to degree 5) are staged in shared memory once; an epilogue thread owns one target and 32
// of the group's slices: per slice one FMA for the grid coordinate, one 24-byte polynomial lookup (the lanes of a
// warp read the same slice's table), one degree-5 Horner.  The four partial sums of a target (32 slices each) are
// added in shared memory and the group's sum goes to the target's fp64 accumulator with one atomic.
constexpr int FE_T = 128;          // targets per tile (UMMA M)
constexpr int FE_S = 128;          // slices per group (UMMA N): each target tile is loaded once per 128 slices
constexpr int FE_STAGES = 2;
constexpr int FE_QCAP = 40;        // cells of interpolation polynomials staged per slice (wider: read from global)
constexpr int FE_EPI = 16;         // epilogue warps: FE_H per TMEM lane quadrant, FE_SPW slices each
constexpr int FE_H = FE_EPI / 4, FE_SPW = FE_S / FE_H;
constexpr int FE_HALF = 16;        // TMEM columns (slices) loaded per round of an epilogue warp
static_assert(FE_SPW % FE_HALF == 0 && FE_HALF % 8 == 0, "TMEM loads of 8 columns");
constexpr int FE_WALLOC = FE_EPI, FE_WTMA = FE_EPI + 2, FE_WMMA = FE_EPI + 3;   // (roles as in k_proj_spread)
constexpr int FE_THREADS = 32 * (4 + FE_EPI);
constexpr int FE_PIECE = FE_T * 128;                      // one k-block of 128 targets: 16 KB
constexpr int FE_B = FE_S * 128;                          // one k-block of the group's directions: 16 KB
constexpr int FE_OFF_STAGE = FS_KBMAX * FE_B;             // 32 KB of resident directions
// the cells' degree-5 polynomials in three planes of coefficient pairs (0-1, 2-3, 4-5), float2 [FE_S][FE_QCAP] each:
// an 8-byte lookup per plane is served in 2 wavefronts (ncu: a 16-byte lookup of the same cells took 5)
constexpr int FE_OFF_Q = FE_OFF_STAGE + FE_STAGES * 2 * FE_PIECE;    // coefficients 0-1 | 2-3 (two planes)
constexpr int FE_OFF_Q1 = FE_OFF_Q + FE_S * FE_QCAP * 16;            // coefficients 4-5
constexpr int FE_OFF_SP = FE_OFF_Q1 + FE_S * FE_QCAP * 8;            // per-slice constants float4 [FE_S]
constexpr int FE_OFF_SPQ = FE_OFF_SP + FE_S * 16;                    // (ga, gb) per slice float2 [FE_S]
constexpr int FE_OFF_SPK = FE_OFF_SPQ + FE_S * 8;                    // 0x4B400000 - 1 + lminA per slice int [FE_S]
constexpr int FE_OFF_RED = FE_OFF_SPK + FE_S * 4;                    // partial sums [2][FE_H][FE_T] fp32
constexpr int FE_OFF_BAR = FE_OFF_RED + 2 * FE_H * FE_T * 4;
constexpr int FE_SMEM = FE_OFF_BAR + 256 + 1024;
static_assert(FE_SMEM <= 227 * 1024, "k_proj_eval shared memory");

// position of cell c in a slice's staged table.  8-byte entries (the planes of coefficient pairs): plain layout --
// ncu counts the ideal 2 wavefronts per warp lookup without a swizzle (measured: the swizzle c ^ ((c >> 4) & 15)
// only cost its instructions)
__device__ __forceinline__ int qswz2(int c) { return c; }

__global__ void __launch_bounds__(FE_THREADS, 1)
    k_proj_eval(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmY,
                const __grid_constant__ CUtensorMap tmYlo, int nk, int klast, int64_t M,
                int np, int ranges, const float* __restrict__ rs, const float* __restrict__ inv_norm,
                const FPar* __restrict__ fp,
                const float* __restrict__ Q, int ncap, int w, double* __restrict__ s64,
                const unsigned* __restrict__ flag16) {
  if (call_failed(flag16)) return;
  extern __shared__ unsigned char feraw[];
  // aligned by pointer arithmetic on the __shared__ array (shared state space kept: LDS / STS)
  unsigned char* sm = feraw + ((1024u - (smem_u32(feraw) & 1023u)) & 1023u);
  float2* sqa = reinterpret_cast<float2*>(sm + FE_OFF_Q);                     // [FE_S][FE_QCAP]: coefficients 0-1
  float2* sqb = reinterpret_cast<float2*>(sm + FE_OFF_Q + FE_S * FE_QCAP * 8);  // 2-3
  float2* sq1 = reinterpret_cast<float2*>(sm + FE_OFF_Q1); // [FE_S][FE_QCAP]: coefficients 4-5 (6, 7: economised)
  float4* sp = reinterpret_cast<float4*>(sm + FE_OFF_SP);  // (ga, gb, -, -) per slice; .z = int bits of lminA, .w = WQ
  float* red = reinterpret_cast<float*>(sm + FE_OFF_RED);  // [2][FE_H][FE_T]
  // the staged-table path reads the slice constants of 4 slices with two 16-byte and one 16-byte broadcast
  // (3 wavefronts) instead of four (one per slice)
  float2* spq = reinterpret_cast<float2*>(sm + FE_OFF_SPQ);
  int* spk = reinterpret_cast<int*>(sm + FE_OFF_SPK);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(sm + FE_OFF_BAR);
  uint64_t* xfull = bfull + 1;
  uint64_t* empty = xfull + FE_STAGES;
  uint64_t* tfull = empty + FE_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ngroups = (np + FE_S - 1) / FE_S;
  const int g = blockIdx.x % ngroups, r = blockIdx.x / ngroups;
  const int s0 = g * FE_S;
  const int64_t ntt = (M + FE_T - 1) / FE_T;
  const int64_t t0 = r * ntt / ranges, t1 = (r + 1) * ntt / ranges;
  const int64_t qs = q_stride(ncap);

  // the group's per-slice constants and interpolation polynomials (all threads)
  for (int ls = threadIdx.x; ls < FE_S; ls += FE_THREADS) {
    const int p = s0 + ls;
    float4 c = make_float4(0.f, 0.f, __int_as_float(0), __int_as_float(1));   // (dead slice: cell 0 of a zero table)
    if (p < np) {
      const FPar f = fp[p];
      const float taun = f.tau * static_cast<float>(1 << f.logn);
      c = make_float4(inv_norm[p] * taun, -fmaf(f.cen, taun, 0.5f * w), __int_as_float(f.lminA), __int_as_float(f.WA));
    }
    sp[ls] = c;
    spq[ls] = make_float2(c.x, c.y);
    spk[ls] = 0x4B400000 - 1 + __float_as_int(c.z);   // cell of a = (bits of floor(a) + 1.5 2^23) - spk
  }
  // (two planes: the lanes of a warp read one slice's table at ~16 distinct cells; 16- and 8-byte cell strides)
  for (int e = threadIdx.x; e < FE_S * FE_QCAP; e += FE_THREADS) {
    const int ls = e / FE_QCAP, cell = e - ls * FE_QCAP;
    const int p = s0 + ls;
    float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 v1 = make_float2(0.f, 0.f);
    if (p < np && cell < fp[p].WA) {
      const float4* qc = reinterpret_cast<const float4*>(Q + p * qs + cell * 8);
      v0 = __ldg(qc);
      const float4 hi = __ldg(qc + 1);
      v1 = make_float2(hi.x, hi.y);
    }
    sqa[ls * FE_QCAP + qswz2(cell)] = make_float2(v0.x, v0.y);
    sqb[ls * FE_QCAP + qswz2(cell)] = make_float2(v0.z, v0.w);
    sq1[ls * FE_QCAP + qswz2(cell)] = v1;
  }
  if (warp == 0 && lane == 0) {
    mbar_init(bfull, 1);
    for (int s = 0; s < FE_STAGES; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], FE_EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmY)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmYlo)) : "memory");
  }
  if (warp == FE_WALLOC) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * FE_S));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == FE_WTMA && lane == 0) {
    // ---- TMA producer: the group's directions (fp16 x 2^8) once, then the target tiles' fp16 hi and lo pieces
    mbar_expect_tx(bfull, nk * FE_B);
    for (int kb = 0; kb < nk; ++kb) tma_load_2d(&tmB, bfull, sm + kb * FE_B, kb * 64, s0);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = t0; t < t1; ++t)
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* sa = sm + FE_OFF_STAGE + stage * 2 * FE_PIECE;
        mbar_expect_tx(&xfull[stage], 2 * FE_PIECE);
        tma_load_2d(&tmY, &xfull[stage], sa, kb * 64, static_cast<int>(t * FE_T));
        tma_load_2d(&tmYlo, &xfull[stage], sa + FE_PIECE, kb * 64, static_cast<int>(t * FE_T));
        if (++stage == FE_STAGES) { stage = 0; phase ^= 1; }
      }
  } else if (warp == FE_WMMA && lane == 0) {
    // ---- MMA issuer: D[target][slice] += A (s_t y: hi, then lo) . B (2^8 g, fp16-exact), K = 16 per MMA
    constexpr uint32_t idesc = idesc_f16(FE_T, FE_S);
    mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int b = it & 1;
      mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(b * FE_S);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&xfull[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned char* sa = sm + FE_OFF_STAGE + stage * 2 * FE_PIECE;
        const uint64_t db = umma_desc_sw128(sm + kb * FE_B);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint64_t da = umma_desc_sw128(sa + q * FE_PIECE);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (kb == nk - 1 && k >= klast) break;   // (k-steps wholly in the zero padding beyond d)
            const uint32_t acc = (kb > 0 || q > 0 || k > 0) ? 1u : 0u;
            const uint64_t adv = static_cast<uint64_t>((k * 32) >> 4);
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                "l"(da + adv), "l"(db + adv), "r"(idesc), "r"(acc));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[stage]))
                     : "memory");
        if (++stage == FE_STAGES) { stage = 0; phase ^= 1; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&tfull[b]))
                   : "memory");
    }
  } else if (warp < FE_EPI) {
    // ---- epilogue: warp w owns TMEM lane quadrant q = w % 4 (targets 32 q + lane of the tile) and the FE_SPW
    //      slices h = w / 4 of the group
    const int q = warp & 3, h = warp >> 2;
    bool fits = true;   // (warp-uniform) every table of the warp's slices is staged in shared memory
    for (int j = 0; j < FE_SPW; ++j) fits &= __float_as_int(sp[FE_SPW * h + j].w) <= FE_QCAP;
    int it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int b = it & 1;
      const float rt = __ldg(rs + 16 * t + 4 * q + (lane >> 3));   // this target's 1 / (2^8 s_g): exact
      mbar_wait_sleep(&tfull[b], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr =
          tmem_base + static_cast<uint32_t>(b * FE_S + FE_SPW * h) + (static_cast<uint32_t>(32 * q) << 16);
      float acc = 0.f;
#pragma unroll 1
      for (int hf = 0; hf < FE_SPW; hf += FE_HALF) {   // FE_HALF columns per TMEM load round: few registers held
        uint32_t v[FE_HALF];
#pragma unroll
        for (int j8 = 0; j8 < FE_HALF; j8 += 8)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=r"(v[j8]), "=r"(v[j8 + 1]), "=r"(v[j8 + 2]), "=r"(v[j8 + 3]), "=r"(v[j8 + 4]),
                         "=r"(v[j8 + 5]), "=r"(v[j8 + 6]), "=r"(v[j8 + 7])
                       : "r"(taddr + hf + j8));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (hf + FE_HALF == FE_SPW) {   // the accumulator is read: release it to the MMAs of tile t + 2
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
        if (fits) {
          // every table of the warp's slices is staged: 4 slices at a time, their cells and both table loads first,
          // then the 4 Horner chains (independent: latency hidden by ILP).  Dead slices (p >= np) have a zero table
          // and WA = 1: they add exactly 0
#pragma unroll
          for (int j0 = 0; j0 < FE_HALF; j0 += 4) {
            float fr[4];
            float4 c0[4];
            float2 c1[4];
            const int lq = FE_SPW * h + hf + j0;   // (a multiple of 4)
            const float4 g01 = reinterpret_cast<const float4*>(spq)[lq / 2];       // broadcasts
            const float4 g23 = reinterpret_cast<const float4*>(spq)[lq / 2 + 1];
            const int4 kq = reinterpret_cast<const int4*>(spk)[lq / 4];
            const float gav[4] = {g01.x, g01.z, g23.x, g23.z}, gbv[4] = {g01.y, g01.w, g23.y, g23.w};
            const int kv[4] = {kq.x, kq.y, kq.z, kq.w};
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int ls = lq + jj;
              const float a = fmaf(__uint_as_float(v[j0 + jj]), gav[jj] * rt, gbv[jj]), fl = floorf(a);
              fr[jj] = a - fl;
              // (fl is an integer of magnitude < 2^22: its int value from the 1.5 2^23 shift, no F2I)
              int cl = __float_as_int(fl + 12582912.f) - kv[jj];
              SKS_CHECK(t * FE_T + 32 * q + lane >= M || s0 + ls >= np || (cl >= 0 && cl < __float_as_int(sp[ls].w)));
              // (memory safety only: every staged table is zero beyond its WA <= FE_QCAP cells)
              cl = cl < 0 ? 0 : (cl >= FE_QCAP ? FE_QCAP - 1 : cl);
              const float2 qa = sqa[ls * FE_QCAP + qswz2(cl)], qb = sqb[ls * FE_QCAP + qswz2(cl)];
              c0[jj] = make_float4(qa.x, qa.y, qb.x, qb.y);
              c1[jj] = sq1[ls * FE_QCAP + qswz2(cl)];
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              float tv = fmaf(c1[jj].y, fr[jj], c1[jj].x);
              tv = fmaf(tv, fr[jj], c0[jj].w);
              tv = fmaf(tv, fr[jj], c0[jj].z);
              tv = fmaf(tv, fr[jj], c0[jj].y);
              acc += fmaf(tv, fr[jj], c0[jj].x);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < FE_HALF; ++j) {
            const int ls = FE_SPW * h + hf + j;
            const float4 c = sp[ls];   // broadcast
            const float a = fmaf(__uint_as_float(v[j]), c.x * rt, c.y), fl = floorf(a);
            int cl = static_cast<int>(fl) + 1 - __float_as_int(c.z);
            const int wq = __float_as_int(c.w);
            SKS_CHECK(t * FE_T + 32 * q + lane >= M || s0 + ls >= np || (cl >= 0 && cl < wq));   // the bound holds
            cl = cl < 0 ? 0 : (cl >= wq ? wq - 1 : cl);   // (a valid bound never clamps; memory safety only)
            float4 c0;
            float2 c1;
            if (wq <= FE_QCAP) {
              const float2 qa = sqa[ls * FE_QCAP + qswz2(cl)], qb = sqb[ls * FE_QCAP + qswz2(cl)];
              c0 = make_float4(qa.x, qa.y, qb.x, qb.y);
              c1 = sq1[ls * FE_QCAP + qswz2(cl)];
            } else {   // footprint wider than the staged table: the polynomial from global memory
              const float4* qp = reinterpret_cast<const float4*>(Q + (s0 + ls) * qs + cl * 8);
              c0 = __ldg(qp);
              const float4 hi = __ldg(qp + 1);
              c1 = make_float2(hi.x, hi.y);
            }
            const float fr = a - fl;
            float tv = fmaf(c1.y, fr, c1.x);
            tv = fmaf(tv, fr, c0.w);
            tv = fmaf(tv, fr, c0.z);
            tv = fmaf(tv, fr, c0.y);
            tv = fmaf(tv, fr, c0.x);
            acc += (s0 + ls < np) ? tv : 0.f;
          }
        }
      }
      float* rb = red + (b * FE_H) * FE_T;
      rb[h * FE_T + 32 * q + lane] = acc;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * FE_H) : "memory");   // the quadrant's partial sums
      if (h == 0) {
        const int64_t m = t * FE_T + 32 * q + lane;
        double sum = 0.0;
#pragma unroll
        for (int hh = 0; hh < FE_H; ++hh) sum += static_cast<double>(rb[hh * FE_T + 32 * q + lane]);
        if (m < M) atomicAdd(s64 + m, sum);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == FE_WALLOC) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * FE_S));
}

// 2-byte elements (fp16), 64 per 128-byte swizzled row of the box
bool encode_h16_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                    uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int fused_dp16(int d) { return (d + 7) / 8 * 8; }

size_t source_bound_bytes(int d) { return sizeof(double) * static_cast<size_t>(d) * (1 + MEAN_PARTS) + 32; }

bool fused_spread_ok(int d, const float* x) {
  return d <= 64 * FS_KBMAX && d % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
}

cudaError_t launch_source_mean(const float* x, int64_t N, int d, double* mu, unsigned* nb, cudaStream_t st) {
  double* part = mu + d;   // [MEAN_PARTS][d] scratch after mu (source_bound_bytes)
  k_sample_mean_part<<<MEAN_PARTS, 128, 0, st>>>(x, N, d, part);
  k_sample_mean_fin<<<1, 128, 0, st>>>(N, d, part, mu, nb);
  return cudaGetLastError();
}

cudaError_t launch_source_prep(const float* x, int64_t N, const float* y, int64_t M, int d, const double* mu,
                               unsigned* nb, uint16_t* xh, uint16_t* xl, float* rsx, uint16_t* yh, uint16_t* yl,
                               float* rsy, const float* w, float* wpad, cudaStream_t st) {
  const int dp16 = fused_dp16(d);
  auto prep = [&](const float* z, int64_t n, unsigned* out, uint16_t* h, uint16_t* l, float* rs, const float* w,
                  float* wp) {
    int64_t blocks = ((n + 127) / 128 * (128 / PR_G) + 7) / 8;
    if (blocks > 148 * 4) blocks = 148 * 4;
    k_prep_f16<<<static_cast<unsigned>(blocks), 256, 0, st>>>(z, n, d, dp16, mu, out,
                                                                       reinterpret_cast<__half*>(h),
                                                                       reinterpret_cast<__half*>(l), rs, w, wp);
  };
  prep(x, N, nb, xh, xl, rsx, w, wpad);
  prep(y, M, nb + 4, yh, yl, rsy, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_bound_ranges(const float* g32, int dp32, int d, const float* inv_norm, int np, const double* mu,
                                const unsigned* nb, unsigned* mm, unsigned* flag16, cudaStream_t st) {
  k_bound_ranges<<<(np + 7) / 8, 256, 0, st>>>(g32, dp32, d, inv_norm, np, mu, nb, 1, mm, flag16);
  return cudaGetLastError();
}

cudaError_t launch_proj_spread(const uint16_t* xh, const uint16_t* xl, const float* rsx, int64_t N, int d,
                               const uint16_t* g16, int dpg, const float* inv_norm, int np, const float* wpad,
                               const FPar* fp, const PolyWin& pw, int ncap, float* grid, const unsigned* flag16,
                               cudaStream_t st) {
  CUtensorMap tmA, tmX, tmXlo;
  const int dp16 = fused_dp16(d), nk = (d + 63) / 64, klast = (d - 64 * (nk - 1) + 15) / 16;
  if (!encode_h16_map(&tmA, g16, static_cast<uint64_t>(np), static_cast<uint64_t>(dpg), static_cast<uint64_t>(dpg),
                      FS_S) ||
      !encode_h16_map(&tmX, xh, static_cast<uint64_t>(N), static_cast<uint64_t>(dp16), static_cast<uint64_t>(dp16),
                      FS_P) ||
      !encode_h16_map(&tmXlo, xl, static_cast<uint64_t>(N), static_cast<uint64_t>(dp16), static_cast<uint64_t>(dp16),
                      FS_P))
    return cudaErrorInvalidValue;
  const int ntiles_s = (np + FS_S - 1) / FS_S;
  const int64_t ntp = (N + FS_P - 1) / FS_P;
  int ranges = 148 / ntiles_s;
  if (ranges < 1) ranges = 1;
  if (ranges > ntp) ranges = static_cast<int>(ntp);
  auto go = [&](auto kern) {
    set_smem_attr_once(reinterpret_cast<const void*>(kern), FS_SMEM);
    kern<<<ntiles_s * ranges, FS_THREADS, FS_SMEM, st>>>(tmA, tmX, tmXlo, nk, klast, N, np, ranges, rsx, inv_norm,
                                                         wpad, fp, pw, ncap, grid, flag16);
  };
  // all variants (see k_proj_spread): each slice tile runs in the one its footprints select
  constexpr int NA = FS_NCOL, NB = FS_EPI / 4;
  switch (pw.w) {
    case 4: go(k_proj_spread<4, NA>); go(k_proj_spread<4, NB>); go(k_proj_spread<4, 1>); break;
    case 5: go(k_proj_spread<5, NA>); go(k_proj_spread<5, NB>); go(k_proj_spread<5, 1>); break;
    case 6: go(k_proj_spread<6, NA>); go(k_proj_spread<6, NB>); go(k_proj_spread<6, 1>); break;
    case 7: go(k_proj_spread<7, NA>); go(k_proj_spread<7, NB>); go(k_proj_spread<7, 1>); break;
    case 8: go(k_proj_spread<8, NA>); go(k_proj_spread<8, NB>); go(k_proj_spread<8, 1>); break;
    case 10: go(k_proj_spread<10, NA>); go(k_proj_spread<10, NB>); go(k_proj_spread<10, 1>); break;
    case 12: go(k_proj_spread<12, NA>); go(k_proj_spread<12, NB>); go(k_proj_spread<12, 1>); break;
    default: return cudaErrorInvalidValue;   // (widths 9, 11: the unfused path)
  }
  return cudaGetLastError();
}

cudaError_t launch_proj_eval(const uint16_t* yh, const uint16_t* yl, const float* rsy, int64_t M, int d,
                             const uint16_t* g16, int dpg, const float* inv_norm, int np, const FPar* fp,
                             const float* Q, int ncap, int w, double* s64, const unsigned* flag16, cudaStream_t st) {
  CUtensorMap tmB, tmY, tmYlo;
  const int dp16 = fused_dp16(d), nk = (d + 63) / 64, klast = (d - 64 * (nk - 1) + 15) / 16;
  if (!encode_h16_map(&tmB, g16, static_cast<uint64_t>(np), static_cast<uint64_t>(dpg), static_cast<uint64_t>(dpg),
                      FE_S) ||
      !encode_h16_map(&tmY, yh, static_cast<uint64_t>(M), static_cast<uint64_t>(dp16), static_cast<uint64_t>(dp16),
                      FE_T) ||
      !encode_h16_map(&tmYlo, yl, static_cast<uint64_t>(M), static_cast<uint64_t>(dp16), static_cast<uint64_t>(dp16),
                      FE_T))
    return cudaErrorInvalidValue;
  const int ngroups = (np + FE_S - 1) / FE_S;
  const int64_t ntt = (M + FE_T - 1) / FE_T;
  int ranges = 148 / ngroups;
  if (ranges < 1) ranges = 1;
  if (ranges > ntt) ranges = static_cast<int>(ntt);
  set_smem_attr_once(reinterpret_cast<const void*>(k_proj_eval), FE_SMEM);
  k_proj_eval<<<ngroups * ranges, FE_THREADS, FE_SMEM, st>>>(tmB, tmY, tmYlo, nk, klast, M, np, ranges, rsy, inv_norm,
                                                            fp, Q, ncap, w, s64, flag16);
  return cudaGetLastError();
}

}  // namespace sks
