// ndft.cu -- rows a5 + a7 by the non-equispaced DFT on the kept band (Sec. 3.1): the engine the
// paper itself uses for the Gaussian.  With the slice's torus scaling u = tau_p (z - cen_p) in
// [-1/2, 1/2) (reading R3) and the band k_lo <= |k| <= k_hi (R5):
//     what_k = sum_n w_n e^{-2 pi i k u_n}                                  (F^H_{C,x} w,  P:508-509)
//     t_m    = sum_{|k| in band} c_k what_k e^{2 pi i k u_m}
//            = [k_lo = 0] c_0 what_0 + 2 sum_{k>0} c_k Re(what_k e^{2 pi i k u_m})   (c_k real and even, w real)
// No window and no grid: the only approximation is the band truncation of the periodised counterpart.  The
// cost per point is K complex rotations and multiply-adds (K = k_hi - k_lo + 1), all in registers, so for the
// narrow Gaussian bands of high-dimensional data (K ~ 10-20, e.g. BJ cfg3 / cfg5) it undercuts the NFFT's
// w taps x polynomial window + shared-memory gridding.  Sums over points: fp32 per thread, fp64 across CTAs.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace sks {

namespace {

constexpr int ND_T = 256;

template <int KW>
__global__ void __launch_bounds__(ND_T) k_ndft_spread(ZView zv, const float* __restrict__ w, const FPar* __restrict__ fp,
                                                      int64_t chunk, double* __restrict__ what,
                                                      const unsigned* __restrict__ flag16) {
  __shared__ float red[ND_T / 32][2 * KW];
  if (call_failed(flag16)) return;
  const int p = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const FPar f = fp[p];
  const int klo = f.klo;
  const float* zx = zv.zx + p * zv.ldx;
  const int64_t i0 = blockIdx.x * chunk, i1 = min(zv.N, i0 + chunk);
  float are[KW], aim[KW];
#pragma unroll
  for (int k = 0; k < KW; ++k) { are[k] = 0.f; aim[k] = 0.f; }
  for (int64_t i = i0 + tid; i < i1; i += ND_T) {
    const float u = __fmul_rn(__fsub_rn(__ldg(zx + i), f.cen), f.tau);
    const float wi = __ldg(w + i);
    float s1, c1, s0, c0;
    sincospif(2.0f * u, &s1, &c1);                               // e^{-2 pi i u} = c1 - i s1
    sincospif(2.0f * static_cast<float>(klo) * u, &s0, &c0);     // e^{-2 pi i k_lo u}
    float cr = wi * c0, ci = -wi * s0;                             // w e^{-2 pi i k u}, k = k_lo
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      are[k] += cr;
      aim[k] += ci;
      const float nr = fmaf(cr, c1, ci * s1);                      // * (c1 - i s1)
      ci = fmaf(ci, c1, -cr * s1);
      cr = nr;
    }
  }
  // CTA reduction: warps by shuffles, then across warps in shared memory; fp64 atomics across CTAs
#pragma unroll
  for (int k = 0; k < KW; ++k) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      are[k] += __shfl_xor_sync(0xffffffffu, are[k], o);
      aim[k] += __shfl_xor_sync(0xffffffffu, aim[k], o);
    }
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < KW; ++k) { red[wid][2 * k] = are[k]; red[wid][2 * k + 1] = aim[k]; }
  __syncthreads();
  if (tid < 2 * KW) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < ND_T / 32; ++q) s += red[q][tid];
    atomicAdd(what + static_cast<int64_t>(p) * 2 * KW + tid, s);
  }
}

// per target: one sincos pair per slice, then K rotations and multiply-adds; slices of a group share the
// coefficients c_k what_k (shared memory), targets vary fastest in the grid
constexpr int NE_T = 256, NE_SG = 32;

template <int KW>
__global__ void __launch_bounds__(NE_T) k_ndft_eval(ZView zv, int np, const FPar* __restrict__ fp,
                                                    const float* __restrict__ D, int dstride,
                                                    const double* __restrict__ what, TargetAcc tacc,
                                                    float* __restrict__ per_slice_out, bool accumulate_out,
                                                    const unsigned* __restrict__ flag16) {
  __shared__ float2 ch[NE_SG][KW];   // (2 - [k = 0]) c_k what_k
  __shared__ float2 pc[NE_SG];       // (tau, cen)
  __shared__ int plo[NE_SG];
  if (call_failed(flag16)) return;
  const int p0 = blockIdx.y * NE_SG, p1 = min(np, p0 + NE_SG);
  for (int e = threadIdx.x; e < (p1 - p0) * KW; e += NE_T) {
    const int q = e / KW, k = e - q * KW;
    const int p = p0 + q;
    const FPar f = fp[p];
    const int klo = f.klo, khi = f.khi;
    const int kk = klo + k;
    float2 v = make_float2(0.f, 0.f);
    if (kk <= khi) {
      const double c = static_cast<double>(D[static_cast<int64_t>(p) * dstride + kk]) * (kk == 0 ? 1.0 : 2.0);
      const double* wp = what + static_cast<int64_t>(p) * 2 * KW + 2 * k;
      v = make_float2(static_cast<float>(c * wp[0]), static_cast<float>(c * wp[1]));
    }
    ch[q][k] = v;
    if (k == 0) { pc[q] = make_float2(f.tau, f.cen); plo[q] = klo; }
  }
  __syncthreads();
  const int64_t m = blockIdx.x * static_cast<int64_t>(NE_T) + threadIdx.x;
  if (m >= zv.M) return;
  double acc = 0.0;
  for (int p = p0; p < p1; ++p) {
    const int q = p - p0;
    const float u = __fmul_rn(__fsub_rn(__ldg(zv.zy + p * zv.ldy + m), pc[q].y), pc[q].x);
    float s1, c1, s0, c0;
    sincospif(2.0f * u, &s1, &c1);                                 // e^{+2 pi i u} = c1 + i s1
    sincospif(2.0f * static_cast<float>(plo[q]) * u, &s0, &c0);
    float cr = c0, ci = s0, t0 = 0.f, t1 = 0.f;
#pragma unroll
    for (int k = 0; k < KW; k += 2) {
      const float2 a = ch[q][k];
      t0 = fmaf(a.x, cr, fmaf(-a.y, ci, t0));                       // Re(a e^{i k theta})
      float nr = fmaf(cr, c1, -ci * s1);
      ci = fmaf(ci, c1, cr * s1);
      cr = nr;
      const float2 b = ch[q][k + 1];
      t1 = fmaf(b.x, cr, fmaf(-b.y, ci, t1));
      nr = fmaf(cr, c1, -ci * s1);
      ci = fmaf(ci, c1, cr * s1);
      cr = nr;
    }
    const float t = t0 + t1;
    if (per_slice_out) {
      float* o = per_slice_out + static_cast<int64_t>(p) * zv.M + m;
      *o = accumulate_out ? *o + t : t;
    }
    acc += t;
  }
  acc_target(tacc, blockIdx.y, m, acc);
}

}  // namespace

cudaError_t launch_ndft_spread(ZView zv, const float* w, int np, const FPar* fp, double* what, bool det,
                               const unsigned* flag16, cudaStream_t st) {
  if (zv.N == 0) return cudaSuccess;
  int64_t chunk = 16384;
  while (chunk > 1024 && ((zv.N + chunk - 1) / chunk) * np < 4 * 148) chunk >>= 1;
  if (det) chunk = zv.N;   // deterministic mode: one CTA per slice, no cross-CTA atomics
  const unsigned nchunk = static_cast<unsigned>((zv.N + chunk - 1) / chunk);
  k_ndft_spread<kNdftWidth><<<dim3(nchunk, np), ND_T, 0, st>>>(zv, w, fp, chunk, what, flag16);
  return cudaGetLastError();
}

static_assert(kNdftEvalGroup == NE_SG, "deterministic groups of the NDFT eval");

cudaError_t launch_ndft_eval(ZView zv, int np, const FPar* fp, const float* D, int dstride, const double* what,
                             TargetAcc acc, float* per_slice_out, bool accumulate_out, const unsigned* flag16,
                             cudaStream_t st) {
  const unsigned bx = static_cast<unsigned>((zv.M + NE_T - 1) / NE_T);
  const unsigned by = static_cast<unsigned>((np + NE_SG - 1) / NE_SG);
  k_ndft_eval<kNdftWidth><<<dim3(bx, by), NE_T, 0, st>>>(zv, np, fp, D, dstride, what, acc, per_slice_out,
                                                         accumulate_out, flag16);
  return cudaGetLastError();
}

}  // namespace sks
