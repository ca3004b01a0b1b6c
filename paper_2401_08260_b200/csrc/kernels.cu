// kernels.cu -- sm_100a kernels of libsks: ranges / prologue helpers and the NFFT path.
//
// Row map (SURVEY.md Sec. 8a / DESIGN.md):
//   a1 projection ............ proj_tc.cu           (Alg.1)
//   a2 torus plan (D_k) ....... k_plan_D             (R3-R7b)
//   a3 sort + a4 scans/evaluate: sortpart.cu (owner-partitioned counting sort, fp64 prefix sums; Sec. 3.2, Alg. 2)
//   a5 spread ................. k_spread_private / k_spread_shared   (NFFT adjoint)
//   a6 FFT x D iFFT ........... k_fft_filter
//   a7 interpolate + mean ..... k_eval (Fourier part) + k_finalize   (Alg.1)
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <tuple>

#include "kernels.h"

namespace sks {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned f2key(float f) {  // order-preserving float -> uint
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float key2f(unsigned k) {
  unsigned u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

void set_smem_attr_once(const void* kernel, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert(std::make_tuple(kernel, dev, bytes)).second)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void decode_minmax(const unsigned* enc, float* dec, int n) {
  for (int i = 0; i < n; ++i) dec[i] = key2f(enc[i]);
}

// bucket index: monotone non-decreasing in z (fp32 sub/mul round monotonically), clamped to [0, nb)
__device__ __forceinline__ int bucket_of(float z, float zmin, float scale, int nb) {
  float t = __fmul_rn(__fsub_rn(z, zmin), scale);
  int b = (t >= 0.f) ? static_cast<int>(t) : 0;   // t < 2^31 guaranteed by min()
  return b < nb ? b : nb - 1;
}

// all w tap weights of a point with fractional offset f by Horner (FMA-only, no MUFU)  (R6)
template <int WT>
__device__ __forceinline__ void poly_taps(const PolyWin& pw, float f, float* out) {
#pragma unroll
  for (int j = 0; j < WT; ++j) {
    const float* c = pw.c + j * (PW_D + 1);
    float acc = c[PW_D];
#pragma unroll
    for (int k = PW_D - 1; k >= 0; --k) acc = fmaf(acc, f, c[k]);
    out[j] = acc;
  }
}

// all w tap weights from the centered even / odd form: a pair of mirror taps costs 3 + 3 + 2 FMA (vs 2 x 7)
template <int WT>
__device__ __forceinline__ void poly_taps_eo(const PolyWin& pw, float f, float* out) {
  const float u = f - 0.5f, u2 = u * u;
#pragma unroll
  for (int j = 0; j < WT / 2; ++j) {
    const float* e = pw.eo[j];
    const float E = fmaf(fmaf(fmaf(e[3], u2, e[2]), u2, e[1]), u2, e[0]);
    const float O = fmaf(fmaf(fmaf(e[7], u2, e[6]), u2, e[5]), u2, e[4]);
    out[j] = fmaf(u, O, E);
    out[WT - 1 - j] = fmaf(-u, O, E);
  }
  if (WT & 1) {   // middle tap of an odd window
    const float* e = pw.eo[WT / 2];
    const float E = fmaf(fmaf(fmaf(e[3], u2, e[2]), u2, e[1]), u2, e[0]);
    const float O = fmaf(fmaf(fmaf(e[7], u2, e[6]), u2, e[5]), u2, e[4]);
    out[WT / 2] = fmaf(u, O, E);
  }
}

// grid coordinate: identical fp32 op sequence on host (planner footprint) and device
__device__ __forceinline__ float grid_coord(float z, float cen, float tau, float nf) {
  return __fmul_rn(__fmul_rn(__fsub_rn(z, cen), tau), nf);
}

__global__ void k_init_minmax(unsigned* mm, int np) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) { mm[i * 4 + 0] = 0xffffffffu; mm[i * 4 + 1] = 0u; mm[i * 4 + 2] = 0xffffffffu; mm[i * 4 + 3] = 0u; }
}

__global__ void k_minmax(ZView zv, unsigned* mm, int* flag) {
  const int p = blockIdx.y;
  float xmn = CUDART_INF_F, xmx = -CUDART_INF_F, amn = CUDART_INF_F, amx = -CUDART_INF_F;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < zv.N + zv.M; i += (int64_t)gridDim.x * blockDim.x) {
    const float z = (i < zv.N) ? zv.zx[p * zv.ldx + i] : zv.zy[p * zv.ldy + (i - zv.N)];
    if (!isfinite(z)) bad = true;
    amn = fminf(amn, z);
    amx = fmaxf(amx, z);
    if (i < zv.N) { xmn = fminf(xmn, z); xmx = fmaxf(xmx, z); }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    xmn = fminf(xmn, __shfl_xor_sync(0xffffffffu, xmn, o));
    xmx = fmaxf(xmx, __shfl_xor_sync(0xffffffffu, xmx, o));
    amn = fminf(amn, __shfl_xor_sync(0xffffffffu, amn, o));
    amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
  }
  if (bad) atomicOr(flag, 1);
  if ((threadIdx.x & 31) == 0) {
    if (xmn <= xmx) { atomicMin(&mm[p * 4 + 0], f2key(xmn)); atomicMax(&mm[p * 4 + 1], f2key(xmx)); }
    if (amn <= amx) { atomicMin(&mm[p * 4 + 2], f2key(amn)); atomicMax(&mm[p * 4 + 3], f2key(amx)); }
  }
}

// call prologue in one launch: zero the flag words, initialise the plan summary, zero the fp64 target sums and
// initialise the first batch's ranges
__global__ void k_prologue(uint4* flag16, double* s64, int64_t M, unsigned* mm, int np) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t == 0) *flag16 = make_uint4(0, 0, 0, 0);
  // the device planner's summary words (flag16 + 4): maxima from 0, minima (k_lo, tau) from all ones
  if (t < kPlanSummaryWords)
    reinterpret_cast<unsigned*>(flag16)[4 + t] = (t == 2 || t == 5) ? 0xffffffffu : 0u;
  if (t < np) { mm[t * 4 + 0] = 0xffffffffu; mm[t * 4 + 1] = 0u; mm[t * 4 + 2] = 0xffffffffu; mm[t * 4 + 3] = 0u; }
  if (s64)
    for (int64_t m = t; m < M; m += static_cast<int64_t>(gridDim.x) * blockDim.x) s64[m] = 0.0;
}

cudaError_t launch_prologue(void* flag16, double* s64, int64_t M, unsigned* mm, int np, cudaStream_t st) {
  int64_t blocks = (std::max<int64_t>(s64 ? M : 0, np) + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_prologue<<<static_cast<unsigned>(blocks), 256, 0, st>>>(static_cast<uint4*>(flag16), s64, M, mm, np);
  return cudaGetLastError();
}

__global__ void k_rerun_prep(unsigned* flag16, unsigned* mm, int np) {
  if (flag16[0] == 0) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    mm[i * 4 + 0] = 0xffffffffu; mm[i * 4 + 1] = 0u; mm[i * 4 + 2] = 0xffffffffu; mm[i * 4 + 3] = 0u;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    flag16[3] = 1u;
    flag16[0] = 0u;
  }
}

cudaError_t launch_rerun_prep(unsigned* flag16, unsigned* mm, int np, cudaStream_t st) {
  k_rerun_prep<<<1, 256, 0, st>>>(flag16, mm, np);   // one CTA: its flag reset follows its range resets
  return cudaGetLastError();
}

cudaError_t launch_init_minmax(unsigned* mm, int np, cudaStream_t st) {
  k_init_minmax<<<(np + 255) / 256, 256, 0, st>>>(mm, np);
  return cudaGetLastError();
}

cudaError_t launch_minmax(ZView zv, int np, unsigned* mm, int* flag, cudaStream_t st) {
  const int64_t L = zv.N + zv.M;
  int bx = static_cast<int>((L + 255) / 256);
  if (bx > 64) bx = 64;
  k_minmax<<<dim3(bx, np), 256, 0, st>>>(zv, mm, flag);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a5: spreading (adjoint NFFT gridding)
// One kernel, the path chosen per slice (uniform per CTA) from the plan's footprint W_p:
//  * W_p <= SP_WMAX_PRIV: per-lane private sub-grids [warp][cell][lane] over the slice's footprint (conflict-free
//    read-modify-writes, no atomics), reduced over warps and lanes at the end;
//  * wider (e.g. the Laplacian's smooth part): one shared grid of n_p cells per CTA.  Shared-memory float atomics
//    are CAS loops on sm_100a, so the CTA accumulates in 32-bit fixed point with native integer atomics, in sub-
//    chunks of SP_SUB points: scale S = 2^30 / sum_{sub-chunk} |w| bounds every partial cell sum by 2^30; the
//    rounding per contribution is <= sum_{sub-chunk} |w| 2^-31, ~1e-9 of the sub-chunk's weight.
// One CTA = (chunk of points, slice).
constexpr int SP_THREADS = 256, SP_WARPS = SP_THREADS / 32, SP_WMAX_PRIV = 64, SP_SUB = 8192;
constexpr int SP_SMEM = SP_WARPS * SP_WMAX_PRIV * 32 * 4;   // = 16384 * 4: also the widest shared grid
static_assert(SP_SMEM >= 16384 * 4, "the shared-grid path needs n_cap floats");

template <int WT>
__device__ __forceinline__ void spread_private(const FPar& f, const float* zx, const float* wc, int cnt, int W,
                                               float nf, const PolyWin& pw, float* priv, float* gp, int n) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float* mine = priv + static_cast<int64_t>(wid) * W * 32;
  for (int c = lane; c < W * 32; c += 32) mine[c] = 0.f;
  __syncwarp();
  const float hw = 0.5f * pw.w;
  float* base = mine - f.lmin * 32 + lane;   // cell l of this lane's private grid: base[l * 32]
  if (pw.w == WT && (WT & 1) == 0) {
    // centered even/odd taps with the coefficients held in registers for the whole loop, four points per
    // iteration.  The coefficients pass through shared memory: read from the constant bank, ptxas would
    // re-load them (and move uniform registers into vector ones) inside the loop
    __shared__ float eos[WT / 2][8];
    if (tid < WT / 2 * 8) eos[tid / 8][tid % 8] = pw.eo[tid / 8][tid % 8];
    __syncthreads();
    float E[WT / 2][4], O[WT / 2][4];
#pragma unroll
    for (int j = 0; j < WT / 2; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        E[j][k] = eos[j][k];
        O[j][k] = eos[j][4 + k];
      }
    const float taun = f.tau * nf;   // nf = 2^k: ((z - cen) tau) nf == (z - cen) (tau nf) exactly (grid_coord)
    auto one = [&](float z, float wi) {
      const float a = __fsub_rn(__fmul_rn(__fsub_rn(z, f.cen), taun), hw), fl = floorf(a);
      const float u = (a - fl) - 0.5f, u2 = u * u;
      SKS_CHECK(static_cast<int>(fl) + 1 - f.lmin >= 0 && static_cast<int>(fl) + 1 - f.lmin + WT <= W);
      float* cell = base + (static_cast<int>(fl) + 1) * 32;
#pragma unroll
      for (int j = 0; j < WT / 2; ++j) {
        const float Ej = fmaf(fmaf(fmaf(E[j][3], u2, E[j][2]), u2, E[j][1]), u2, E[j][0]);
        const float Oj = fmaf(fmaf(fmaf(O[j][3], u2, O[j][2]), u2, O[j][1]), u2, O[j][0]);
        cell[j * 32] = fmaf(wi, fmaf(u, Oj, Ej), cell[j * 32]);
        cell[(WT - 1 - j) * 32] = fmaf(wi, fmaf(-u, Oj, Ej), cell[(WT - 1 - j) * 32]);
      }
    };
    int i0 = 0;
    if (((reinterpret_cast<uintptr_t>(zx) | reinterpret_cast<uintptr_t>(wc)) & 15) == 0) {
      // four consecutive points per thread by 16-byte loads (coalesced, all four in flight)
      for (; i0 + 4 * SP_THREADS <= cnt; i0 += 4 * SP_THREADS) {
        const float4 z = __ldg(reinterpret_cast<const float4*>(zx + i0) + tid);
        const float4 ww = __ldg(reinterpret_cast<const float4*>(wc + i0) + tid);
        one(z.x, ww.x);
        one(z.y, ww.y);
        one(z.z, ww.z);
        one(z.w, ww.w);
      }
    }
    for (int i = i0 + tid; i < cnt; i += SP_THREADS) one(__ldg(zx + i), __ldg(wc + i));
  } else {
    for (int i = tid; i < cnt; i += SP_THREADS) {
      const float v = grid_coord(__ldg(zx + i), f.cen, f.tau, nf);
      const float a = __fsub_rn(v, hw), fl = floorf(a);
      const float wi = __ldg(wc + i);
      float tw[WT];
      poly_taps<WT>(pw, a - fl, tw);                  // generic WT = 12 kernel for other widths
      SKS_CHECK(static_cast<int>(fl) + 1 - f.lmin >= 0 && static_cast<int>(fl) + 1 - f.lmin + pw.w <= W);
      float* cell = base + (static_cast<int>(fl) + 1) * 32;
#pragma unroll
      for (int j = 0; j < WT; ++j) cell[j * 32] += wi * tw[j];
    }
  }
  __syncthreads();
  // reduce: cell c -> sum over warps (registers) then lanes (shuffles)
  for (int c = wid; c < W; c += SP_WARPS) {
    float s = 0.f;
#pragma unroll 8
    for (int q = 0; q < SP_WARPS; ++q) s += priv[(static_cast<int64_t>(q) * W + c) * 32 + lane];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && s != 0.f) atomicAdd(&gp[(f.lmin + c) & (n - 1)], s);
  }
}

template <int WT>
__device__ __forceinline__ void spread_shared(const FPar& f, const float* zx, const float* wc, int cnt, float nf,
                                              const PolyWin& pw, int* sgi, float* gp, int n) {
  __shared__ float wred[SP_THREADS / 32];
  const int tid = threadIdx.x;
  const float hw = 0.5f * pw.w;
  for (int s0 = 0; s0 < cnt; s0 += SP_SUB) {
    const int s1 = min(cnt, s0 + SP_SUB);
    for (int c = tid; c < n; c += SP_THREADS) sgi[c] = 0;
    float aw = 0.f;
    for (int i = s0 + tid; i < s1; i += SP_THREADS) aw += fabsf(__ldg(wc + i));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) aw += __shfl_xor_sync(0xffffffffu, aw, o);
    if ((tid & 31) == 0) wred[tid >> 5] = aw;
    __syncthreads();
    float wsum = 0.f;
#pragma unroll
    for (int q = 0; q < SP_THREADS / 32; ++q) wsum += wred[q];
    if (wsum > 0.f) {   // (uniform: all weights of this sub-chunk zero otherwise)
      const float S = 1073741824.0f / (wsum * 1.0001f);   // 2^30 / sum|w| (margin for the fp32 sum)
      for (int i = s0 + tid; i < s1; i += SP_THREADS) {
        const float v = grid_coord(__ldg(zx + i), f.cen, f.tau, nf);
        const float a = __fsub_rn(v, hw), fl = floorf(a);
        const int l0 = static_cast<int>(fl) + 1;
        const float ws = __ldg(wc + i) * S;
        float tw[WT];
        poly_taps<WT>(pw, a - fl, tw);
#pragma unroll
        for (int j = 0; j < WT; ++j) atomicAdd(&sgi[(l0 + j) & (n - 1)], __float2int_rn(ws * tw[j]));
      }
      __syncthreads();
      const float inv = 1.0f / S;
      for (int c = tid; c < n; c += SP_THREADS) {
        const int v = sgi[c];
        if (v != 0) atomicAdd(&gp[c], static_cast<float>(v) * inv);
      }
    }
    __syncthreads();
  }
}

// a grid larger than the launch's shared-memory capacity (rare: a slice whose plan needs n_p beyond it): the taps
// go straight to the global grid with atomics
template <int WT>
__device__ __forceinline__ void spread_global(const FPar& f, const float* zx, const float* wc, int cnt, float nf,
                                              const PolyWin& pw, float* gp, int n) {
  const float hw = 0.5f * pw.w;
  for (int i = threadIdx.x; i < cnt; i += SP_THREADS) {
    const float v = grid_coord(__ldg(zx + i), f.cen, f.tau, nf);
    const float a = __fsub_rn(v, hw), fl = floorf(a);
    const int l0 = static_cast<int>(fl) + 1;
    const float wi = __ldg(wc + i);
    float tw[WT];
    poly_taps<WT>(pw, a - fl, tw);
#pragma unroll
    for (int j = 0; j < WT; ++j) atomicAdd(&gp[(l0 + j) & (n - 1)], wi * tw[j]);
  }
}

// cap: the launch's shared memory in floats.  Per slice: private sub-grids if they fit (W * 8 warps * 32 lanes),
// else a fixed-point shared grid if n_p fits, else global atomics
template <int WT>
__global__ void __launch_bounds__(SP_THREADS) k_spread(ZView zv, const float* __restrict__ w,
                                                       const FPar* __restrict__ fp, int ncap, PolyWin pw,
                                                       int64_t chunk, float* __restrict__ grid, int cap,
                                                       const unsigned* __restrict__ flag16) {
  extern __shared__ float spsm[];
  if (call_failed(flag16)) return;
  const int p = blockIdx.y;
  const FPar f = fp[p];
  const int n = 1 << f.logn;
  const float nf = static_cast<float>(n);
  const int64_t i0 = blockIdx.x * chunk;
  const int cnt = static_cast<int>(min(zv.N, i0 + chunk) - i0);   // 32-bit loop inside the chunk
  const float* zx = zv.zx + p * zv.ldx + i0;
  const float* wc = w + i0;
  float* gp = grid + static_cast<int64_t>(p) * ncap;
  if (f.W <= SP_WMAX_PRIV && f.W * SP_WARPS * 32 <= cap) spread_private<WT>(f, zx, wc, cnt, f.W, nf, pw, spsm, gp, n);
  else if (n <= cap) spread_shared<WT>(f, zx, wc, cnt, nf, pw, reinterpret_cast<int*>(spsm), gp, n);
  else spread_global<WT>(f, zx, wc, cnt, nf, pw, gp, n);
}

cudaError_t launch_spread(ZView zv, const float* w, int np, const FPar* fp, int ncap, const PolyWin& pw,
                          bool wide_likely, bool det, float* grid, const unsigned* flag16, cudaStream_t st) {
  // chunking: enough CTAs to fill 148 SMs several times, >= 2048 points per CTA to amortise the flush (narrow
  // footprints: up to 32768 points per CTA; wide ones (the Laplacian) flush n_p cells per 8192-point sub-chunk).
  // Deterministic mode: the whole slice in one CTA (its grid cells are then written by one thread each, in order)
  int64_t chunk = wide_likely ? 8192 : 32768;
  while (chunk > 2048 && ((zv.N + chunk - 1) / chunk) * np < (wide_likely ? 4 : 16) * 148) chunk >>= 1;
  if (det) chunk = zv.N;
  const unsigned nchunk = static_cast<unsigned>((zv.N + chunk - 1) / chunk);
  if (nchunk == 0) return cudaSuccess;
  // shared memory: 32 KB -- private sub-grids up to 32 cells (the Gaussian footprints of BJ cfg3 / cfg5: 17 / 31),
  // a shared grid of up to 8192 cells (the Laplacian's n_p ~ 4096) -- keeps 7 CTAs per SM (64 KB: 3; measured
  // cfg4 spread 0.35 -> 0.23 ms)
  const int smem = SP_SMEM / 2;
  auto go = [&](auto kern) {
    set_smem_attr_once(reinterpret_cast<const void*>(kern), smem);
    kern<<<dim3(nchunk, np), SP_THREADS, smem, st>>>(zv, w, fp, ncap, pw, chunk, grid, smem / 4, flag16);
  };
  switch (pw.w) {
    case 4: go(k_spread<4>); break;
    case 6: go(k_spread<6>); break;
    case 8: go(k_spread<8>); break;
    default: go(k_spread<12>); break;   // taps beyond w have zero coefficients
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a6: FFT -> x D -> inverse FFT (one CTA per slice)
constexpr int FF_THREADS = 512;

// radix-2 stages.  PS: tw holds one contiguous twiddle table per stage (stage s: e^{-2 pi i pos / 2^s} at
// tw[2^(s-1) - 1 + pos], n - 1 entries), so consecutive lanes read consecutive twiddles (no bank conflicts);
// otherwise (n = 16384, shared memory) the n/2 twiddles of the last stage, read with stride n / 2^s
template <bool PS>
__device__ __forceinline__ void fft_stages(float2* buf, const float2* tw, int n, int logn) {
  for (int s = 1; s <= logn; ++s) {
    const int half = 1 << (s - 1);
    const float2* tws = PS ? tw + (half - 1) : tw;
    const int tstride = PS ? 1 : (n >> s);
    for (int b = threadIdx.x; b < n / 2; b += FF_THREADS) {
      const int grp = b >> (s - 1), pos = b & (half - 1);
      const int i = grp * 2 * half + pos, j = i + half;
      const float2 t = tws[pos * tstride];
      const float2 a = buf[i], c = buf[j];
      const float2 bt = make_float2(c.x * t.x - c.y * t.y, c.x * t.y + c.y * t.x);
      buf[i] = make_float2(a.x + bt.x, a.y + bt.y);
      buf[j] = make_float2(a.x - bt.x, a.y - bt.y);
    }
    __syncthreads();
  }
}

// one launch per capacity tier: this launch handles the slices with nlo < n_p <= cap (its shared memory holds
// cap complex cells and their twiddles), the others exit at once
__global__ void __launch_bounds__(FF_THREADS) k_fft_filter(const float* __restrict__ grid, const float* __restrict__ D,
                                                           int ncap, const FPar* __restrict__ fp, PolyWin pw,
                                                           float* __restrict__ Q, int nlo, int cap, int econ,
                                                           const unsigned* __restrict__ flag16) {
  extern __shared__ float2 sm[];
  if (call_failed(flag16)) return;
  const int p = blockIdx.x;
  const FPar f = fp[p];
  const int logn = f.logn, n = 1 << logn;
  if (n <= nlo || n > cap) return;
  float2* buf = sm;          // [n]
  float2* tw = sm + cap;     // per-stage forward twiddles (fft_stages)
  const bool ps = n <= 8192;
  if (ps) {
    for (int j = threadIdx.x; j < n - 1; j += FF_THREADS) {
      const int half = 1 << (31 - __clz(j + 1)), pos = j + 1 - half;   // stage with 2^(s-1) = half
      float sv, cv;
      sincospif(static_cast<float>(pos) / static_cast<float>(half), &sv, &cv);   // angle 2 pi pos / (2 half)
      tw[j] = make_float2(cv, -sv);
    }
  } else {
    for (int j = threadIdx.x; j < n / 2; j += FF_THREADS) {
      float sv, cv;
      sincospif(2.0f * static_cast<float>(j) / static_cast<float>(n), &sv, &cv);
      tw[j] = make_float2(cv, -sv);
    }
  }
  const float* gp = grid + static_cast<int64_t>(p) * ncap;
  for (int l = threadIdx.x; l < n; l += FF_THREADS) buf[__brev(l) >> (32 - logn)] = make_float2(gp[l], 0.f);
  __syncthreads();
  if (ps) fft_stages<true>(buf, tw, n, logn);      // G_k = sum_l g_l e^{-2 pi i k l / n}
  else fft_stages<false>(buf, tw, n, logn);
  const float* Dp = D + static_cast<int64_t>(p) * (ncap / 2 + 1);
  for (int k = threadIdx.x; k < n; k += FF_THREADS) {
    const float dk = Dp[k <= n / 2 ? k : n - k];
    const float2 v = buf[k];
    buf[k] = make_float2(v.x * dk, -v.y * dk);      // conj(D_k G_k)
  }
  __syncthreads();
  for (int l = threadIdx.x; l < n; l += FF_THREADS) {   // bit-reversal permutation in place
    const int r = __brev(l) >> (32 - logn);
    if (l < r) { const float2 t = buf[l]; buf[l] = buf[r]; buf[r] = t; }
  }
  __syncthreads();
  if (ps) fft_stages<true>(buf, tw, n, logn);      // h_l = conj(FFT(conj X))_l; real part
  else fft_stages<false>(buf, tw, n, logn);
  // interpolation polynomials of the footprint cells: Q[c][k] = sum_j h[lminA + c + j] coef_j[k]
  const int l00 = f.lminA, WA = f.WA;
  float* qp = Q + static_cast<int64_t>(p) * q_stride(ncap);
  if (!econ) {
    for (int e = threadIdx.x; e < WA * (PW_D + 1); e += FF_THREADS) {
      const int c = e / (PW_D + 1), k = e - c * (PW_D + 1);
      float acc = 0.f;
      for (int j = 0; j < pw.w; ++j) acc = fmaf(buf[(l00 + c + j) & (n - 1)].x, pw.c[j * (PW_D + 1) + k], acc);
      qp[e] = acc;
    }
    return;
  }
  // economised to degree 5 (the fused interpolation reads 6 coefficients per cell): one thread per cell forms the
  // degree-7 polynomial in fp64, then subtracts (a_7 / 2^13) T*_7 and (a_6 / 2^11) T*_6 (shifted Chebyshev
  // polynomials T*_n(f) = T_n(2 f - 1), leading coefficient 2^(2n-1)): the change is at most |a_7| / 2^13 + |a_6'| /
  // 2^11 on f in [0, 1] (|T*_n| <= 1) -- 0.5-2e-6 of the cell's amplitude for a band within n_p / 4 (R6b)
  static_assert(PW_D == 7, "economisation of degree-7 polynomials");
  for (int c = threadIdx.x; c < WA; c += FF_THREADS) {
    double a[PW_D + 1];
#pragma unroll
    for (int k = 0; k <= PW_D; ++k) a[k] = 0.0;
    for (int j = 0; j < pw.w; ++j) {
      const double hv = buf[(l00 + c + j) & (n - 1)].x;
#pragma unroll
      for (int k = 0; k <= PW_D; ++k) a[k] = fma(hv, static_cast<double>(pw.c[j * (PW_D + 1) + k]), a[k]);
    }
    const double t7[8] = {-1.0, 98.0, -1568.0, 9408.0, -26880.0, 39424.0, -28672.0, 8192.0};
    const double t6[7] = {1.0, -72.0, 840.0, -3584.0, 6912.0, -6144.0, 2048.0};
    const double r7 = a[7] / 8192.0;
#pragma unroll
    for (int k = 0; k <= 7; ++k) a[k] -= r7 * t7[k];
    const double r6 = a[6] / 2048.0;
#pragma unroll
    for (int k = 0; k <= 6; ++k) a[k] -= r6 * t6[k];
#pragma unroll
    for (int k = 0; k <= PW_D; ++k) qp[c * (PW_D + 1) + k] = k <= 5 ? static_cast<float>(a[k]) : 0.f;
  }
}

cudaError_t launch_fft_filter(const float* grid, const float* D, int np, int ncap, const FPar* fp, const PolyWin& pw,
                              float* Q, int cap_hint, bool econ, const unsigned* flag16, cudaStream_t st) {
  // two capacity tiers: the common grids (n_p <= cap_hint) with the shared memory they need -- several CTAs per SM
  // -- and, predicated on the device plan, any larger grid up to n_cap in a second launch whose CTAs otherwise exit
  auto smem_for = [](int cap) {
    return static_cast<size_t>(cap) * sizeof(float2) + static_cast<size_t>(cap <= 8192 ? cap : cap / 2) * sizeof(float2);
  };
  set_smem_attr_once(reinterpret_cast<const void*>(k_fft_filter), static_cast<int>(smem_for(ncap)));
  // (at most one CTA per SM anyway -- np <= 148 -- one launch at full capacity saves the second launch's latency)
  const int cap = np <= 148 ? ncap : std::min(cap_hint, ncap);
  k_fft_filter<<<np, FF_THREADS, smem_for(cap), st>>>(grid, D, ncap, fp, pw, Q, 0, cap, econ ? 1 : 0, flag16);
  if (cap < ncap)
    k_fft_filter<<<np, FF_THREADS, smem_for(ncap), st>>>(grid, D, ncap, fp, pw, Q, cap, ncap, econ ? 1 : 0, flag16);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a7: interpolation at the targets
// grid (target blocks, slice groups): each thread handles one target over EV_SG slices, then one fp64
// atomic into s64 (or per-slice stores for sks_sum_1d).  Target blocks vary fastest, so the CTAs resident
// at a time work on the same slice group and its polynomials stay in L2.  A target's value on slice p is one
// degree-7 Horner on the interpolation polynomial of its cell (Q, written by k_fft_filter).
constexpr int EV_THREADS = 256, EV_SG = 32;

__device__ __forceinline__ float horner8(float4 c0, float4 c1, float fr) {
  float t = fmaf(c1.w, fr, c1.z);
  t = fmaf(t, fr, c1.y);
  t = fmaf(t, fr, c1.x);
  t = fmaf(t, fr, c0.w);
  t = fmaf(t, fr, c0.z);
  t = fmaf(t, fr, c0.y);
  return fmaf(t, fr, c0.x);
}

__device__ __forceinline__ double eval_one(const EvalArgs& a, int p, float z, float hw, int64_t m, int64_t M) {
  const double zd = z;
  double t = 0.0;
  const FPar f = a.fp[p];
  if (a.moment) {
    const SliceTot T = a.tot[p];
    t += a.mom_coef * static_cast<double>(f.tau) * (T.C - 2.0 * zd * T.B + zd * zd * T.A);
  }
  if (a.fourier) {
    const float v = grid_coord(z, f.cen, f.tau, static_cast<float>(1 << f.logn));
    const float av = __fsub_rn(v, hw), fl = floorf(av);
    const int l0 = static_cast<int>(fl) + 1;
    static_assert(PW_D == 7, "interpolation polynomials are read as two float4");
    SKS_CHECK(l0 - f.lminA >= 0 && l0 - f.lminA < f.WA);
    const float4* q = reinterpret_cast<const float4*>(a.Q + static_cast<int64_t>(p) * q_stride(a.ncap) +
                                                      (l0 - f.lminA) * 8);
    t += horner8(__ldg(q), __ldg(q + 1), av - fl);
  }
  if (a.per_slice_out) {
    float* o = a.per_slice_out + static_cast<int64_t>(p) * M + m;
    *o = a.accumulate_out ? *o + static_cast<float>(t) : static_cast<float>(t);
  }
  return t;
}

__global__ void __launch_bounds__(EV_THREADS) k_eval(EvalArgs a) {
  if (call_failed(a.flag16)) return;
  const int64_t M = a.zv.M;
  const int64_t m = blockIdx.x * static_cast<int64_t>(EV_THREADS) + threadIdx.x;
  if (m >= M) return;
  const int p0 = blockIdx.y * EV_SG, p1 = min(a.np, p0 + EV_SG);
  const float hw = 0.5f * a.w;
  double acc = 0.0;
  int p = p0;
  for (; p + 4 <= p1; p += 4) {   // 4 independent slices in flight per target
    float z[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) z[k] = __ldg(a.zv.zy + (p + k) * a.zv.ldy + m);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += eval_one(a, p + k, z[k], hw, m, M);
  }
  for (; p < p1; ++p) acc += eval_one(a, p, __ldg(a.zv.zy + p * a.zv.ldy + m), hw, m, M);
  acc_target(a.acc, blockIdx.y, m, acc);
}

// the common case (fp64 target sums, no per-slice output): slice parameters staged in shared memory, the cell's 8
// coefficients by one 256-bit load, fp32 partial sums over EV_U slices
constexpr int EV_U = 8;
__device__ __forceinline__ void ld_q8(const float* q, float4& c0, float4& c1) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(c0.x), "=f"(c0.y), "=f"(c0.z), "=f"(c0.w), "=f"(c1.x), "=f"(c1.y), "=f"(c1.z), "=f"(c1.w)
      : "l"(q));
}

template <bool MOMENT>
__global__ void __launch_bounds__(EV_THREADS) k_eval_q(EvalArgs a, int sg) {
  __shared__ float4 sp[EV_SG];   // (cen, tau n_p, Q offset of cell 0 (int bits), -)
  __shared__ double4 st[MOMENT ? EV_SG : 1];   // (sum w, sum w z, sum w z^2, mom_coef tau) (fp64)
  if (call_failed(a.flag16)) return;
  const int p0 = blockIdx.y * sg, p1 = min(a.np, p0 + sg);
  const float hw = 0.5f * a.w;
  const int64_t qs = q_stride(a.ncap);
  for (int q = threadIdx.x; q < p1 - p0; q += EV_THREADS) {
    const FPar f = a.fp[p0 + q];
    // cell l0 = floor(v - w/2) + 1 of slice p reads Q[p][l0 - lminA]: float offset qs (p - p0) + 8 (l0 - lminA)
    const int qoff = static_cast<int>(qs * q) + 8 * (1 - f.lminA);
    sp[q] = make_float4(f.cen, f.tau * static_cast<float>(1 << f.logn), __int_as_float(qoff), __int_as_float(f.WA));
    if (MOMENT) {
      const SliceTot T = a.tot[p0 + q];
      st[q] = make_double4(T.A, T.B, T.C, a.mom_coef * static_cast<double>(f.tau));
    }
  }
  __syncthreads();
  const int64_t m = blockIdx.x * static_cast<int64_t>(EV_THREADS) + threadIdx.x;
  if (m >= a.zv.M) return;
  const float* zy = a.zv.zy + m;
  const float* Qg = a.Q + qs * p0;
  auto one = [&](int q, float z) {
    const float4 c = sp[q];
    const float av = __fsub_rn(__fmul_rn(__fsub_rn(z, c.x), c.y), hw), fl = floorf(av);
    float4 c0, c1;
    SKS_CHECK(__float_as_int(c.z) + 8 * static_cast<int>(fl) >= static_cast<int>(qs) * q &&
              __float_as_int(c.z) + 8 * static_cast<int>(fl) < static_cast<int>(qs) * q + 8 * __float_as_int(c.w));
    ld_q8(Qg + (__float_as_int(c.z) + 8 * static_cast<int>(fl)), c0, c1);
    return horner8(c0, c1, av - fl);
  };
  double acc = 0.0;
  int p = p0;
  // EV_U independent slices in flight per target; the projections of the next EV_U slices are loaded before the
  // current ones are evaluated (the kernel is bound by the latency of the z -> coefficient load chain)
  float zn[EV_U];
  if (p + EV_U <= p1)
#pragma unroll
    for (int k = 0; k < EV_U; ++k) zn[k] = __ldcs(zy + (p + k) * a.zv.ldy);
  for (; p + EV_U <= p1; p += EV_U) {
    float z[EV_U];
#pragma unroll
    for (int k = 0; k < EV_U; ++k) z[k] = zn[k];
    if (p + 2 * EV_U <= p1)
#pragma unroll
      for (int k = 0; k < EV_U; ++k) zn[k] = __ldcs(zy + (p + EV_U + k) * a.zv.ldy);
    float part = 0.f;
#pragma unroll
    for (int k = 0; k < EV_U; ++k) part += one(p - p0 + k, z[k]);
    acc += part;
    if (MOMENT)
#pragma unroll
      for (int k = 0; k < EV_U; ++k) {
        const double zd = z[k];
        const double4 T = st[p - p0 + k];
        acc += T.w * (T.z - 2.0 * zd * T.y + zd * zd * T.x);
      }
  }
  for (; p < p1; ++p) {
    const float z = __ldcs(zy + p * a.zv.ldy);
    acc += one(p - p0, z);
    if (MOMENT) {
      const double zd = z;
      const double4 T = st[p - p0];
      acc += T.w * (T.z - 2.0 * zd * T.y + zd * zd * T.x);
    }
  }
  acc_target(a.acc, blockIdx.y, m, acc);
}

static_assert(kEvalGroup == EV_SG, "deterministic groups of the eval kernels");

cudaError_t launch_eval(const EvalArgs& a, bool det, cudaStream_t st) {
  const unsigned bx = static_cast<unsigned>((a.zv.M + EV_THREADS - 1) / EV_THREADS);
  if (a.fourier && (a.acc.s64 || a.acc.part) && !a.per_slice_out) {
    // slices per CTA: EV_SG, or fewer (down to EV_U) when the targets alone give too few CTAs (small, latency-bound
    // problems such as BJ cfg1: more CTAs in flight at the cost of one more fp64 atomic per target and group; not
    // in deterministic mode, whose groups are fixed)
    int sg = EV_SG;
    while (!det && sg > EV_U && static_cast<int64_t>(bx) * ((a.np + sg - 1) / sg) < 2 * 148) sg >>= 1;
    const unsigned by = static_cast<unsigned>((a.np + sg - 1) / sg);
    if (a.moment) k_eval_q<true><<<dim3(bx, by), EV_THREADS, 0, st>>>(a, sg);
    else k_eval_q<false><<<dim3(bx, by), EV_THREADS, 0, st>>>(a, sg);
  } else {
    const unsigned by = static_cast<unsigned>((a.np + EV_SG - 1) / EV_SG);
    k_eval<<<dim3(bx, by), EV_THREADS, 0, st>>>(a);
  }
  return cudaGetLastError();
}

__global__ void k_zero(uint4* p, size_t n16) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

cudaError_t launch_zero(void* p, size_t bytes, cudaStream_t st) {
  // bytes is a multiple of 16 (workspace carving aligns every region to 256 B)
  const size_t n16 = bytes / 16;
  if (n16 == 0) return cudaSuccess;
  size_t blocks = (n16 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_zero<<<static_cast<unsigned>(blocks), 256, 0, st>>>(static_cast<uint4*>(p), n16);
  return cudaGetLastError();
}

__global__ void k_finalize_det(const double* __restrict__ part, int G, int64_t M, double scale,
                               float* __restrict__ s) {
  for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < M;
       m += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < G; ++g) v += part[static_cast<int64_t>(g) * M + m];
    s[m] = static_cast<float>(v * scale);
  }
}

cudaError_t launch_finalize_det(const double* part, int G, int64_t M, double scale, float* s, cudaStream_t st) {
  int64_t blocks = (M + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_finalize_det<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part, G, M, scale, s);
  return cudaGetLastError();
}

__global__ void k_finalize(const double* __restrict__ s64, int64_t M, double scale, float* __restrict__ s) {
  for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < M; m += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s[m] = static_cast<float>(s64[m] * scale);
}

cudaError_t launch_finalize(const double* s64, int64_t M, double scale, float* s, cudaStream_t st) {
  int64_t blocks = (M + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_finalize<<<static_cast<unsigned>(blocks), 256, 0, st>>>(s64, M, scale, s);
  return cudaGetLastError();
}

}  // namespace sks
