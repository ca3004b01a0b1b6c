// sortpath.cu -- the sort path (rows a3 + a4) for the negative distance kernel and the sorting part of the
// Laplacian decomposition: Sec. 3.2 / Alg. 2 computes, exactly,
//     t_m = -c sum_n w_n |x_n - y_m|                                             (c = c_d or alpha c_d)
// by sorting the merged projections and running prefix sums.  Here the sort is a two-level MSD counting
// sort (both levels in shared memory) and the prefix sums are fp64:
//   level 1 (coarse, B1 value buckets over the slice's x range; many CTAs per slice):
//     K1 k_sp_count   per (chunk, slice): coarse histograms of x and y + fp64 coarse sums of w, wz, wz^2
//     K2 k_sp_scan    per slice: chunk offsets, coarse records {A_excl, B_excl, W, Z, offsets}, slice totals
//     K3 k_sp_scatter per (chunk, slice): x -> (z, w), y -> (z, m) in coarse-bucket order
//   level 2 (fine, one CTA per (coarse bucket, slice), everything in shared memory):
//     K4 k_sp_fine    fine counting sort of the bucket's x and y, fp64 fine prefix sums, and for every target
//                     t = -c [ z (A_lo - A_hi) - B_lo + B_hi + sum_{x in its fine bucket} w |x - z| ]
//                     with A/B = sum w / sum w z over the x strictly below (lo) / above (hi) its fine bucket.
// A bucket map b(z) = floor((z - zmin) * scale) computed with explicitly rounded fp32 ops is monotone in z,
// which is all the identity needs (ties contribute |x - z| = 0 on either side).  The host runs the four
// kernels over L2-sized slice sub-batches so that all scratch stays in the 126 MB L2.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace sks {

namespace {

__device__ __forceinline__ float key2f_dev(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ int coarse_of(float z, float zmin, float scale, int B1) {
  const float t = __fmul_rn(__fsub_rn(z, zmin), scale);
  const int b = (t >= 0.f) ? static_cast<int>(fminf(t, 2.0e9f)) : 0;
  return b < B1 ? b : B1 - 1;
}

// fine index inside coarse bucket b1: monotone in z (each fp32 op rounds monotonically)
__device__ __forceinline__ int fine_of(float z, float zmin, float scale, int b1, int F) {
  const float t = __fmul_rn(__fsub_rn(z, zmin), scale);
  const float u = __fmul_rn(__fsub_rn(t, static_cast<float>(b1)), static_cast<float>(F));
  const int f = (u >= 0.f) ? static_cast<int>(fminf(u, 2.0e9f)) : 0;
  return f < F ? f : F - 1;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// exclusive scan of n ints in smem by a CTA of NT threads (NT multiple of 32, <= 1024); returns the total
template <int NT>
__device__ int block_excl_scan(int* a, int n, int* wbuf) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + NT - 1) / NT;
  const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
  int loc = 0;
  for (int i = b0; i < b1; ++i) loc += a[i];
  const int inc = warp_incl_scan(loc);
  if (lane == 31) wbuf[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int v = lane < NT / 32 ? wbuf[lane] : 0;
    const int vi = warp_incl_scan(v);
    if (lane < NT / 32) wbuf[lane] = vi - v;
    if (lane == 31) wbuf[32] = vi;
  }
  __syncthreads();
  int run = wbuf[wid] + inc - loc;
  for (int i = b0; i < b1; ++i) {
    const int c = a[i];
    a[i] = run;
    run += c;
  }
  const int total = wbuf[32];
  __syncthreads();
  return total;
}

constexpr int SP_T = 256;     // threads of K1/K3/K4
constexpr int K2_T = 256;     // threads of K2
constexpr int FINE_CAP = 1024;

// ---------------------------------------------------------------- K1: coarse histograms + coarse fp64 sums
__global__ void __launch_bounds__(SP_T) k_sp_count(SortArgs a) {
  extern __shared__ unsigned char sm1[];
  const int B1 = a.B1;
  double* sums = reinterpret_cast<double*>(sm1);              // [B1][3]
  int* cnt = reinterpret_cast<int*>(sums + 3 * B1);           // [B1][2]
  const int c = blockIdx.x, p = blockIdx.y, tid = threadIdx.x;
  for (int i = tid; i < 3 * B1; i += SP_T) sums[i] = 0.0;
  for (int i = tid; i < 2 * B1; i += SP_T) cnt[i] = 0;
  const float zmin = key2f_dev(a.mm[p * 4 + 0]), zmax = key2f_dev(a.mm[p * 4 + 1]);
  const float range = zmax - zmin;
  const float scale = (range > 0.f) ? static_cast<float>(B1) / range : 0.f;
  if (c == 0 && tid == 0) { a.bpar[p * 2 + 0] = zmin; a.bpar[p * 2 + 1] = scale; }
  __syncthreads();
  const int64_t i0 = static_cast<int64_t>(c) * a.chunk;
  const float* zx = a.zv.zx + p * a.zv.ldx;
  const float* zy = a.zv.zy + p * a.zv.ldy;
  const int64_t xe = min(a.zv.N, i0 + a.chunk), ye = min(a.zv.M, i0 + a.chunk);
  for (int64_t i = i0 + tid; i < xe; i += SP_T) {
    const float z = __ldg(zx + i), w = __ldg(a.w + i);
    const int b = coarse_of(z, zmin, scale, B1);
    const double wz = static_cast<double>(w) * z;
    atomicAdd(&cnt[2 * b], 1);
    atomicAdd(&sums[3 * b + 0], static_cast<double>(w));
    atomicAdd(&sums[3 * b + 1], wz);
    atomicAdd(&sums[3 * b + 2], wz * z);
  }
  for (int64_t i = i0 + tid; i < ye; i += SP_T) atomicAdd(&cnt[2 * coarse_of(__ldg(zy + i), zmin, scale, B1) + 1], 1);
  __syncthreads();
  const int64_t base = (static_cast<int64_t>(p) * a.nchunks + c) * B1;
  for (int b = tid; b < B1; b += SP_T) {
    reinterpret_cast<int2*>(a.ccnt)[base + b] = make_int2(cnt[2 * b], cnt[2 * b + 1]);
    double* s = a.csum + (base + b) * 3;
    s[0] = sums[3 * b];
    s[1] = sums[3 * b + 1];
    s[2] = sums[3 * b + 2];
  }
}

// ---------------------------------------------------------------- K2: per-slice offsets + coarse records
__global__ void __launch_bounds__(K2_T) k_sp_scan(SortArgs a) {
  __shared__ int wi[33];
  __shared__ double wd[3][K2_T / 32];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B1 = a.B1, nc = a.nchunks;
  const int E = B1 / K2_T;   // B1 is a power of two >= 256
  const int b0 = tid * E;
  int2* cc = reinterpret_cast<int2*>(a.ccnt) + static_cast<int64_t>(p) * nc * B1;
  const double* cs = a.csum + static_cast<int64_t>(p) * nc * B1 * 3;
  CoarseRec* cr = a.crec + static_cast<int64_t>(p) * B1;
  // per bucket: chunk-local exclusive offsets (in place) and totals
  int tx = 0, ty = 0;
  double tW = 0.0, tZ = 0.0, tC = 0.0;
  for (int e = 0; e < E; ++e) {
    const int b = b0 + e;
    int rx = 0, ry = 0;
    double W = 0.0, Z = 0.0, C = 0.0;
    for (int c = 0; c < nc; ++c) {
      const int2 v = cc[static_cast<int64_t>(c) * B1 + b];
      cc[static_cast<int64_t>(c) * B1 + b] = make_int2(rx, ry);
      rx += v.x;
      ry += v.y;
      const double* s = cs + (static_cast<int64_t>(c) * B1 + b) * 3;
      W += s[0];
      Z += s[1];
      C += s[2];
    }
    CoarseRec r;
    r.A = 0.0; r.B = 0.0; r.W = W; r.Z = Z;
    r.xoff = 0; r.xcnt = rx; r.yoff = 0; r.ycnt = ry;
    cr[b] = r;
    tx += rx; ty += ry;
    tW += W; tZ += Z; tC += C;
  }
  // block exclusive scans of (x count, y count) and (W, Z); totals
  const int ix = warp_incl_scan(tx), iy = warp_incl_scan(ty);
  const double iW = warp_incl_scan(tW), iZ = warp_incl_scan(tZ), iC = warp_incl_scan(tC);
  __shared__ int wix[K2_T / 32], wiy[K2_T / 32];
  if (lane == 31) { wix[wid] = ix; wiy[wid] = iy; wd[0][wid] = iW; wd[1][wid] = iZ; wd[2][wid] = iC; }
  __syncthreads();
  if (tid == 0) {
    int sx = 0, sy = 0;
    double sW = 0, sZ = 0, sC = 0;
    for (int q = 0; q < K2_T / 32; ++q) {
      const int vx = wix[q], vy = wiy[q];
      const double vW = wd[0][q], vZ = wd[1][q], vC = wd[2][q];
      wix[q] = sx; wiy[q] = sy; wd[0][q] = sW; wd[1][q] = sZ; wd[2][q] = sC;
      sx += vx; sy += vy; sW += vW; sZ += vZ; sC += vC;
    }
    a.tot[p] = SliceTot{sW, sZ, sC, 0.0};
    wi[0] = sx;
  }
  __syncthreads();
  int ox = wix[wid] + ix - tx, oy = wiy[wid] + iy - ty;
  double oW = wd[0][wid] + iW - tW, oZ = wd[1][wid] + iZ - tZ;
  for (int e = 0; e < E; ++e) {
    const int b = b0 + e;
    CoarseRec r = cr[b];
    r.A = oW; r.B = oZ; r.xoff = ox; r.yoff = oy;
    cr[b] = r;
    for (int c = 0; c < nc; ++c) {
      int2 v = cc[static_cast<int64_t>(c) * B1 + b];
      cc[static_cast<int64_t>(c) * B1 + b] = make_int2(v.x + ox, v.y + oy);
    }
    ox += r.xcnt; oy += r.ycnt; oW += r.W; oZ += r.Z;
  }
}

// ---------------------------------------------------------------- K3: scatter into coarse-bucket order
__global__ void __launch_bounds__(SP_T) k_sp_scatter(SortArgs a) {
  extern __shared__ int cur[];   // [B1][2]
  const int B1 = a.B1;
  const int c = blockIdx.x, p = blockIdx.y, tid = threadIdx.x;
  const int64_t base = (static_cast<int64_t>(p) * a.nchunks + c) * B1;
  for (int b = tid; b < B1; b += SP_T) {
    const int2 v = reinterpret_cast<const int2*>(a.ccnt)[base + b];
    cur[2 * b] = v.x;
    cur[2 * b + 1] = v.y;
  }
  __syncthreads();
  const float zmin = a.bpar[p * 2 + 0], scale = a.bpar[p * 2 + 1];
  const int64_t i0 = static_cast<int64_t>(c) * a.chunk;
  const float* zx = a.zv.zx + p * a.zv.ldx;
  const float* zy = a.zv.zy + p * a.zv.ldy;
  float2* xs = a.xs + static_cast<int64_t>(p) * a.zv.N;
  float2* ys = a.ys + static_cast<int64_t>(p) * a.zv.M;
  const int64_t xe = min(a.zv.N, i0 + a.chunk), ye = min(a.zv.M, i0 + a.chunk);
  for (int64_t i = i0 + tid; i < xe; i += SP_T) {
    const float z = __ldg(zx + i);
    const int pos = atomicAdd(&cur[2 * coarse_of(z, zmin, scale, B1)], 1);
    xs[pos] = make_float2(z, __ldg(a.w + i));
  }
  for (int64_t i = i0 + tid; i < ye; i += SP_T) {
    const float z = __ldg(zy + i);
    const int pos = atomicAdd(&cur[2 * coarse_of(z, zmin, scale, B1) + 1], 1);
    ys[pos] = make_float2(z, __int_as_float(static_cast<int>(i)));
  }
}

// ---------------------------------------------------------------- K4: fine level + evaluation
constexpr size_t FINE_SMEM = FINE_CAP * (2 * sizeof(float2) + 2 * sizeof(int) + 2 * sizeof(double) + 2 * sizeof(float));

__global__ void __launch_bounds__(SP_T) k_sp_fine(SortArgs a) {
  extern __shared__ double sm4[];
  double* fA = sm4;
  double* fB = fA + FINE_CAP;
  float2* xsrt = reinterpret_cast<float2*>(fB + FINE_CAP);
  float2* ysrt = xsrt + FINE_CAP;
  int* cx = reinterpret_cast<int*>(ysrt + FINE_CAP);
  int* cy = cx + FINE_CAP;
  float* fW = reinterpret_cast<float*>(cy + FINE_CAP);
  float* fZ = fW + FINE_CAP;
  __shared__ int wbuf[33];
  __shared__ double wdd[2][SP_T / 32];
  const int b1 = blockIdx.x, p = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const CoarseRec r = a.crec[static_cast<int64_t>(p) * a.B1 + b1];
  const int nx = r.xcnt, ny = r.ycnt;
  if (ny == 0) return;
  const SliceTot T = a.tot[p];
  const float zmin = a.bpar[p * 2 + 0], scale = a.bpar[p * 2 + 1];
  const float2* xg = a.xs + static_cast<int64_t>(p) * a.zv.N + r.xoff;
  const float2* yg = a.ys + static_cast<int64_t>(p) * a.zv.M + r.yoff;
  const int64_t M = a.zv.M;
  if (nx > FINE_CAP || ny > FINE_CAP) {
    // oversize coarse bucket (extreme concentration / duplicates): direct sums over the bucket's x's
    const double Ahi = T.A - r.A - r.W, Bhi = T.B - r.B - r.Z;
    for (int j = tid; j < ny; j += SP_T) {
      const float2 e = yg[j];
      const float z = e.x;
      const double zd = z;
      double same = 0.0;
      for (int i = 0; i < nx; ++i) {
        const float2 q = xg[i];
        same += static_cast<double>(q.y) * fabs(static_cast<double>(q.x) - zd);
      }
      const double t = -a.coef * ((zd * r.A - r.B) + (Bhi - zd * Ahi) + same);
      const int64_t m = __float_as_int(e.y);
      if (a.s64) atomicAdd(a.s64 + m, t);
      if (a.per_slice_out) a.per_slice_out[static_cast<int64_t>(p) * M + m] = static_cast<float>(t);
    }
    return;
  }
  int F = 16;
  while (F < nx && F < FINE_CAP) F <<= 1;
  for (int f = tid; f < F; f += SP_T) { cx[f] = 0; cy[f] = 0; }
  __syncthreads();
  for (int i = tid; i < nx; i += SP_T) atomicAdd(&cx[fine_of(xg[i].x, zmin, scale, b1, F)], 1);
  for (int j = tid; j < ny; j += SP_T) atomicAdd(&cy[fine_of(yg[j].x, zmin, scale, b1, F)], 1);
  __syncthreads();
  block_excl_scan<SP_T>(cx, F, wbuf);
  block_excl_scan<SP_T>(cy, F, wbuf);
  for (int i = tid; i < nx; i += SP_T) {
    const float2 e = xg[i];
    xsrt[atomicAdd(&cx[fine_of(e.x, zmin, scale, b1, F)], 1)] = e;
  }
  for (int j = tid; j < ny; j += SP_T) {
    const float2 e = yg[j];
    ysrt[atomicAdd(&cy[fine_of(e.x, zmin, scale, b1, F)], 1)] = e;
  }
  __syncthreads();
  // fine bucket sums (fp64) and exclusive prefix; after the scatter cx[f] = end of fine bucket f
  {
    const int per = (F + SP_T - 1) / SP_T;
    const int f0 = min(F, tid * per), f1 = min(F, f0 + per);
    double lA = 0.0, lB = 0.0;
    for (int f = f0; f < f1; ++f) {
      const int lo = f ? cx[f - 1] : 0, hi = cx[f];
      double W = 0.0, Z = 0.0;
      for (int i = lo; i < hi; ++i) {
        const float2 q = xsrt[i];
        W += q.y;
        Z += static_cast<double>(q.y) * q.x;
      }
      fW[f] = static_cast<float>(W);
      fZ[f] = static_cast<float>(Z);
      fA[f] = W;   // temporarily the bucket sums
      fB[f] = Z;
      lA += W;
      lB += Z;
    }
    const double iA = warp_incl_scan(lA), iB = warp_incl_scan(lB);
    if (lane == 31) { wdd[0][wid] = iA; wdd[1][wid] = iB; }
    __syncthreads();
    if (tid == 0) {
      double sa = 0.0, sb = 0.0;
      for (int q = 0; q < SP_T / 32; ++q) {
        const double va = wdd[0][q], vb = wdd[1][q];
        wdd[0][q] = sa;
        wdd[1][q] = sb;
        sa += va;
        sb += vb;
      }
    }
    __syncthreads();
    double rA = wdd[0][wid] + iA - lA, rB = wdd[1][wid] + iB - lB;
    for (int f = f0; f < f1; ++f) {
      const double W = fA[f], Z = fB[f];
      fA[f] = rA;
      fB[f] = rB;
      rA += W;
      rB += Z;
    }
  }
  __syncthreads();
  // targets in fine-bucket order (lanes share fine buckets: broadcast smem reads)
  for (int j = tid; j < ny; j += SP_T) {
    const float2 e = ysrt[j];
    const float z = e.x;
    const int f = fine_of(z, zmin, scale, b1, F);
    const int lo = f ? cx[f - 1] : 0, hi = cx[f];
    float same = 0.f;
    for (int i = lo; i < hi; ++i) {
      const float2 q = xsrt[i];
      same = fmaf(q.y, fabsf(q.x - z), same);
    }
    const double zd = z;
    const double Alo = r.A + fA[f], Blo = r.B + fB[f];
    const double Ahi = T.A - Alo - fW[f], Bhi = T.B - Blo - fZ[f];
    const double t = -a.coef * ((zd * Alo - Blo) + (Bhi - zd * Ahi) + static_cast<double>(same));
    const int64_t m = __float_as_int(e.y);
    if (a.s64) atomicAdd(a.s64 + m, t);
    if (a.per_slice_out) a.per_slice_out[static_cast<int64_t>(p) * M + m] = static_cast<float>(t);
  }
}

}  // namespace

int sortpath_coarse_buckets(int64_t N) {
  int64_t b = 256;
  while (b < N / 64 && b < 4096) b <<= 1;
  return static_cast<int>(b);
}

cudaError_t launch_sortpath(const SortArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sp_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 32);
    cudaFuncSetAttribute(k_sp_fine, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FINE_SMEM));
    attr = true;
  }
  const dim3 gc(static_cast<unsigned>(a.nchunks), static_cast<unsigned>(a.np));
  k_sp_count<<<gc, SP_T, static_cast<size_t>(a.B1) * 32, st>>>(a);
  k_sp_scan<<<a.np, K2_T, 0, st>>>(a);
  k_sp_scatter<<<gc, SP_T, static_cast<size_t>(a.B1) * 8, st>>>(a);
  k_sp_fine<<<dim3(static_cast<unsigned>(a.B1), static_cast<unsigned>(a.np)), SP_T, FINE_SMEM, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sks
