// sortpath.cu -- the sort path (rows a3 + a4) for the negative distance kernel and the sorting part of the
// Laplacian decomposition.  Sec. 3.2 / Alg. 2 computes, exactly,
//     t_m = -c sum_n w_n |x_n - y_m|                                       (c = c_d, or alpha c_d)
// by sorting the merged projections and running prefix sums.  Here: one thread-block CLUSTER of SP_C CTAs
// per slice performs a one-pass MSD counting sort of both point sets into NB monotone value buckets of the
// slice's x range, fp64 prefix sums over the x buckets, and a bucket-ordered evaluation of the targets:
//     sum_n w_n |x_n - z| = [z A_lo - B_lo] + [B_hi - z A_hi] + sum_{x in z's bucket} w |x - z|
// (A/B = sum w / sum w z over the x in buckets strictly left (lo) / right (hi) of z's bucket).
//
//  P0 granule histograms -> count-balanced bucket map (NB buckets allotted to NG equal-width granules in
//     proportion to their x counts; linear inside a granule) and bucket ownership (balanced by x + y count)
//  P1 each CTA counts its quarter of x and y into local smem bucket histograms
//  P2 bucket ownership balanced by element count (coarse histograms exchanged through DSMEM); every owner
//     sums the C histograms of its buckets (DSMEM reads), scans them, and writes each CTA's scatter cursors
//     back into that CTA's shared memory (DSMEM writes)
//  P3 each CTA scatters its quarter: (z,w) -> xs, (z,m) -> ys, bucket order (smem cursor atomics)
//  P4 owners: fp64 sums of their buckets, exclusive scan (cross-CTA offsets through DSMEM)
//  P5 records {A_excl, B_excl, off, cnt, w, wz}; slice totals
//  P6 owners evaluate their targets in bucket order (lanes share buckets: broadcast loads), fp64 atomics
// Persistent: one cluster per scratch slot (as many as can be co-resident, ~148/SP_C), each walking its
// slices; the slots' scratch (xs, ys, records: ~2 MB each) is reused and stays in L2.
// The bucket map b(z) = floor((z - zmin) * scale) with explicitly rounded fp32 ops is monotone in z, which is
// all the identity needs (ties contribute |x - z| = 0 on either side).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace sks {

namespace {

constexpr int SP_C = 4;            // CTAs per slice (cluster)
constexpr int SP_T = 1024;         // threads per CTA
constexpr int SP_W = SP_T / 32;
constexpr int NB = 8192;           // buckets per slice
constexpr int NG = 256;            // equal-width granules; buckets are allotted to granules by x count

__device__ __forceinline__ float key2f_dev(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// granule of z: t = (z - zmin) * gscale in [0, NG) for z in the x range (clamped outside)
__device__ __forceinline__ float gran_t(float z, float zmin, float gscale) {
  return __fmul_rn(__fsub_rn(z, zmin), gscale);
}

// count-balanced bucket map: granule g owns buckets [gb.x, gb.x + gb.y); inside a granule the map is linear.
// Monotone non-decreasing in z: t is monotone (rounded fp32 ops), floor(t) is monotone, and every bucket of
// granule g precedes every bucket of granule g+1.
__device__ __forceinline__ int bin_of(float z, float zmin, float gscale, const int2* __restrict__ gtab) {
  const float t = gran_t(z, zmin, gscale);
  int g = (t >= 0.f) ? static_cast<int>(fminf(t, 1.0e9f)) : 0;
  g = g < NG ? g : NG - 1;
  const int2 gb = gtab[g];
  if (gb.y == 0) return min(gb.x, NB - 1);
  const float u = __fmul_rn(__fsub_rn(t, static_cast<float>(g)), static_cast<float>(gb.y));
  int f = (u >= 0.f) ? static_cast<int>(fminf(u, 1.0e9f)) : 0;
  f = f < gb.y ? f : gb.y - 1;
  return gb.x + f;
}

__device__ __forceinline__ int gran_of(float z, float zmin, float gscale) {
  const float t = gran_t(z, zmin, gscale);
  const int g = (t >= 0.f) ? static_cast<int>(fminf(t, 1.0e9f)) : 0;
  return g < NG ? g : NG - 1;
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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block exclusive scan of a[0..n) (ints, smem) by all SP_T threads; returns the total
__device__ int block_scan_int(int* a, int n, int* wbuf) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + SP_T - 1) / SP_T;
  const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
  int loc = 0;
  for (int i = b0; i < b1; ++i) loc += a[i];
  const int inc = warp_incl_scan(loc);
  if (lane == 31) wbuf[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int v = wbuf[lane];
    const int vi = warp_incl_scan(v);
    wbuf[lane] = vi - v;
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

struct __align__(16) Shared {
  int hx[NB];          // local x histogram -> scatter cursors
  int hy[NB];          // local y histogram -> scatter cursors
  int ox[NB + 1];      // owner: absolute start of each owned x bucket (index b - lo)
  int oy[NB + 1];
  int2 gtab[NG];       // bucket map: granule -> (first bucket, #buckets)
  int gx[NG];          // local granule counts of x (then: global, all ranks)
  int gxy[NG];         // local granule counts of x + y (work balance)
  int wbuf[34];
  int tot_i[4];
  double tot_d[4];
  double wsd[3][SP_W];
};

__global__ void __cluster_dims__(SP_C, 1, 1) __launch_bounds__(SP_T, 1) k_sortsum(SortArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Shared& S = *reinterpret_cast<Shared*>(smraw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int slot = blockIdx.x / SP_C, nslots = gridDim.x / SP_C;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t N = a.zv.N, M = a.zv.M;
  // persistent: this cluster owns scratch slot `slot` and walks the slices slot, slot + nslots, ...
  BucketRec* rp = a.rec + static_cast<int64_t>(slot) * NB;
  float2* xsp = a.xs + static_cast<int64_t>(slot) * N;
  float2* ysp = a.ys + static_cast<int64_t>(slot) * M;
  constexpr int U = 8;
  const int64_t x0 = N * rank / SP_C, x1 = N * (rank + 1) / SP_C;
  const int64_t y0 = M * rank / SP_C, y1 = M * (rank + 1) / SP_C;

  long long tph[10];
  int nph = 0;
#define PHASE() do { if (a.dbg && tid == 0 && p == slot) tph[nph++] = clock64(); } while (0)
  for (int p = slot; p < a.np; p += nslots) {
    if (a.only_flagged && !a.ovf[p]) continue;   // uniform across the cluster
    PHASE();
    const float* zx = a.zv.zx + p * a.zv.ldx;
    const float* zy = a.zv.zy + p * a.zv.ldy;
    const float zmin = key2f_dev(a.mm[p * 4 + 0]), zmax = key2f_dev(a.mm[p * 4 + 1]);
    const float range = zmax - zmin;
    const float gscale = (range > 0.f) ? static_cast<float>(NG) / range : 0.f;
    if (rank == 0 && tid == 0) { a.bpar[p * 2 + 0] = zmin; a.bpar[p * 2 + 1] = gscale; }

    // ---- P0: granule histograms of my quarter (x; x + y)
    for (int b = tid; b < NB; b += SP_T) { S.hx[b] = 0; S.hy[b] = 0; }
    for (int g = tid; g < NG; g += SP_T) { S.gx[g] = 0; S.gxy[g] = 0; }
    __syncthreads();
    for (int64_t base = x0; base < x1; base += U * SP_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * SP_T < x1) atomicAdd(&S.gx[gran_of(zz[k], zmin, gscale)], 1);
    }
    for (int64_t base = y0; base < y1; base += U * SP_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * SP_T < y1) atomicAdd(&S.gxy[gran_of(zz[k], zmin, gscale)], 1);
    }
    __syncthreads();
    for (int g = tid; g < NG; g += SP_T) S.gxy[g] += S.gx[g];
    cluster.sync();
    // global granule counts (identical in every rank) -> bucket map and ownership
    int own_g0, own_g1;
    {
      __shared__ int gtx[NG], gtxy[NG];
      for (int g = tid; g < NG; g += SP_T) {
        int cx = 0, cxy = 0;
#pragma unroll
        for (int r = 0; r < SP_C; ++r) {
          const Shared* R = cluster.map_shared_rank(&S, r);
          cx += R->gx[g];
          cxy += R->gxy[g];
        }
        gtx[g] = cx;
        gtxy[g] = cxy;
      }
      __syncthreads();
      if (wid == 0) {   // warp-parallel: lane l handles granules [8l, 8l + 8)
        constexpr int PG = NG / 32;
        long long cx = 0, cxy = 0;
        for (int q = 0; q < PG; ++q) { cx += gtx[lane * PG + q]; cxy += gtxy[lane * PG + q]; }
        const long long ix = warp_incl_scan(cx), ixy = warp_incl_scan(cxy);
        const long long total = __shfl_sync(0xffffffffu, ixy, 31);
        long long cum = ix - cx, run = ixy - cxy;
        int prev = (N > 0) ? static_cast<int>((cum * NB) / N) : 0;
        for (int q = 0; q < PG; ++q) {
          const int g = lane * PG + q;
          cum += gtx[g];
          const int next = (N > 0) ? static_cast<int>((cum * NB) / N) : NB;
          S.gtab[g] = make_int2(prev, next - prev);
          prev = next;
          const long long before = run;
          run += gtxy[g];
          for (int r = 1; r < SP_C; ++r)   // boundary r = first granule end with run*C >= total*r
            if (before * SP_C < total * r && run * SP_C >= total * r) S.wbuf[r] = g + 1;
        }
        if (lane == 0) {
          S.wbuf[0] = 0;
          S.wbuf[SP_C] = NG;
          if (total == 0)
            for (int r = 1; r < SP_C; ++r) S.wbuf[r] = NG;
        }
      }
      __syncthreads();
      own_g0 = S.wbuf[rank];
      own_g1 = S.wbuf[rank + 1];
    }
    const int lo = (own_g0 < NG) ? S.gtab[own_g0].x : NB;
    const int hi = (own_g1 < NG) ? S.gtab[own_g1].x : NB;
    const int nown = hi - lo;

    PHASE();
    // ---- P1: bucket histograms of my quarter
    for (int64_t base = x0; base < x1; base += U * SP_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * SP_T < x1) atomicAdd(&S.hx[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
    }
    for (int64_t base = y0; base < y1; base += U * SP_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * SP_T < y1) atomicAdd(&S.hy[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
    }
    cluster.sync();

    PHASE();
    // ---- P2: owners sum the ranks' histograms of their buckets, scan, write every rank's cursors
    for (int j = tid; j < nown; j += SP_T) {
      int tx = 0, ty = 0;
#pragma unroll
      for (int r = 0; r < SP_C; ++r) {
        const Shared* R = cluster.map_shared_rank(&S, r);
        tx += R->hx[lo + j];
        ty += R->hy[lo + j];
      }
      S.ox[j] = tx;
      S.oy[j] = ty;
    }
    __syncthreads();
    const int Sx = block_scan_int(S.ox, nown, S.wbuf);
    const int Sy = block_scan_int(S.oy, nown, S.wbuf);
    if (tid == 0) { S.tot_i[0] = Sx; S.tot_i[1] = Sy; }
    cluster.sync();
    int bx = 0, by = 0;
    for (int r = 0; r < rank; ++r) {
      const Shared* R = cluster.map_shared_rank(&S, r);
      bx += R->tot_i[0];
      by += R->tot_i[1];
    }
    for (int j = tid; j < nown; j += SP_T) { S.ox[j] += bx; S.oy[j] += by; }
    if (tid == 0) { S.ox[nown] = bx + Sx; S.oy[nown] = by + Sy; }
    __syncthreads();
    for (int j = tid; j < nown; j += SP_T) {
      int rx = S.ox[j], ry = S.oy[j];
#pragma unroll
      for (int r = 0; r < SP_C; ++r) {
        Shared* R = cluster.map_shared_rank(&S, r);
        const int hx = R->hx[lo + j], hy = R->hy[lo + j];
        R->hx[lo + j] = rx;
        R->hy[lo + j] = ry;
        rx += hx;
        ry += hy;
      }
    }
    cluster.sync();

    PHASE();
    // ---- P3: scatter my quarter
    for (int64_t base = x0; base < x1; base += U * SP_T) {
      float zz[U], ww[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
        ww[k] = (i < x1) ? __ldg(a.w + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * SP_T < x1) {
          if (a.variant == 2) {
            atomicAdd(&S.hx[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
            xsp[base + tid + k * SP_T] = make_float2(zz[k], ww[k]);
          } else {
            const int pos = atomicAdd(&S.hx[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
            if (a.variant != 1) xsp[pos] = make_float2(zz[k], ww[k]);
          }
        }
    }
    for (int64_t base = y0; base < y1; base += U * SP_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * SP_T;
        if (i < y1) {
          if (a.variant == 2) {
            atomicAdd(&S.hy[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
            ysp[i] = make_float2(zz[k], __int_as_float(static_cast<int>(i)));
          } else {
            const int pos = atomicAdd(&S.hy[bin_of(zz[k], zmin, gscale, S.gtab)], 1);
            if (a.variant != 1) ysp[pos] = make_float2(zz[k], __int_as_float(static_cast<int>(i)));
          }
        }
      }
    }
    cluster.sync();   // release/acquire at cluster scope: the scattered xs/ys are visible to the owners

    PHASE();
    // ---- P4 + P5: owner bucket sums (thread per run of consecutive buckets, fp64), exclusive scan, records
    const int per = (nown + SP_T - 1) / SP_T;
    const int j0 = min(nown, tid * per), j1 = min(nown, j0 + per);
    double lA = 0.0, lB = 0.0, lC = 0.0;
    for (int i0 = S.ox[j0], i1 = S.ox[j1]; i0 < i1; i0 += 8) {   // 8 loads in flight
      float2 qq[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) qq[u] = (i0 + u < i1) ? __ldcg(xsp + i0 + u) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double wz = static_cast<double>(qq[u].y) * qq[u].x;
        lA += qq[u].y;
        lB += wz;
        lC += wz * qq[u].x;
      }
    }
    {
      const double iA = warp_incl_scan(lA), iB = warp_incl_scan(lB);
      const double sC = warp_sum(lC);
      if (lane == 31) { S.wsd[0][wid] = iA; S.wsd[1][wid] = iB; }
      if (lane == 0) S.wsd[2][wid] = sC;
      __syncthreads();
      if (wid == 0) {
        const double va = S.wsd[0][lane], vb = S.wsd[1][lane], vc = S.wsd[2][lane];
        const double ia = warp_incl_scan(va), ib = warp_incl_scan(vb), sc = warp_sum(vc);
        S.wsd[0][lane] = ia - va;
        S.wsd[1][lane] = ib - vb;
        if (lane == 31) { S.tot_d[0] = ia; S.tot_d[1] = ib; }
        if (lane == 0) S.tot_d[2] = sc;
      }
      cluster.sync();   // owners' partial totals published
      double TA = 0, TB = 0, TC = 0, PA = 0, PB = 0;
#pragma unroll
      for (int r = 0; r < SP_C; ++r) {
        const Shared* R = cluster.map_shared_rank(&S, r);
        TA += R->tot_d[0]; TB += R->tot_d[1]; TC += R->tot_d[2];
        if (r < rank) { PA += R->tot_d[0]; PB += R->tot_d[1]; }
      }
      if (rank == 0 && tid == 0) a.tot[p] = SliceTot{TA, TB, TC, 0.0};
      double rA = PA + S.wsd[0][wid] + iA - lA, rB = PB + S.wsd[1][wid] + iB - lB;
      for (int j = j0; j < j1; ++j) {
        double W = 0.0, Z = 0.0;
        for (int i0 = S.ox[j], i1 = S.ox[j + 1]; i0 < i1; i0 += 8) {
          float2 qq[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) qq[u] = (i0 + u < i1) ? __ldcg(xsp + i0 + u) : make_float2(0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            W += qq[u].y;
            Z += static_cast<double>(qq[u].y) * qq[u].x;
          }
        }
        BucketRec r;
        r.A = rA;
        r.B = rB;
        r.off = S.ox[j];
        r.cnt = S.ox[j + 1] - S.ox[j];
        r.w = static_cast<float>(W);
        r.wz = static_cast<float>(Z);
        rp[lo + j] = r;
        rA += W;
        rB += Z;
      }
      __syncthreads();

      PHASE();
      // ---- P6: my targets in bucket order
      const int t0 = S.oy[0], t1 = S.oy[nown];
      for (int base = t0; base < t1; base += 2 * SP_T) {
        float2 ee[2];
        int bb[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = base + tid + k * SP_T;
          ee[k] = (i < t1) ? __ldcg(ysp + i) : make_float2(zmin, 0.f);
          bb[k] = bin_of(ee[k].x, zmin, gscale, S.gtab);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = base + tid + k * SP_T;
          if (i >= t1) continue;
          const BucketRec R = rp[bb[k]];
          const float z = ee[k].x;
          const int64_t m = __float_as_int(ee[k].y);
          const double zd = z;
          const double Ahi = TA - R.A - R.w, Bhi = TB - R.B - R.wz;
          const float2* xp = xsp + R.off;
          float s0 = 0.f, s1 = 0.f;
          for (int j0c = 0; j0c < R.cnt; j0c += 16) {   // up to 16 bucket entries in flight
            float2 qq[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) qq[u] = (j0c + u < R.cnt) ? __ldcg(xp + j0c + u) : make_float2(z, 0.f);
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
              s0 = fmaf(qq[u].y, fabsf(qq[u].x - z), s0);
              s1 = fmaf(qq[u + 1].y, fabsf(qq[u + 1].x - z), s1);
            }
          }
          const double same = static_cast<double>(s0 + s1);
          const double t = -a.coef * ((zd * R.A - R.B) + (Bhi - zd * Ahi) + same);
          if (a.s64) atomicAdd(a.s64 + m, t);
          if (a.per_slice_out) a.per_slice_out[static_cast<int64_t>(p) * M + m] = static_cast<float>(t);
        }
      }
    }
    PHASE();
    cluster.sync();   // slot scratch and smem are reused by the next slice
  }
  if (a.dbg && tid == 0)
    for (int k = 0; k + 1 < nph; ++k) a.dbg[static_cast<int64_t>(blockIdx.x) * 8 + k] = tph[k + 1] - tph[k];
#undef PHASE
}

// ======================================================================================================
// DSMEM-resident variant (default when a slice fits): a cluster of C = 8 or 16 CTAs per slice; every owner
// CTA keeps ITS buckets' x entries (z, w) and y entries (z, m) in its own shared memory.  The scatter is a
// DSMEM store into the owner, the bucket sums / scans / target evaluation read local shared memory only.
// Local histograms are packed 16-bit x|y counters (one u32 per bucket).  A slice whose owners would exceed
// the capacity (extreme concentration, duplicates) is flagged in a.ovf and done by k_sortsum above.
constexpr int DS_T = 1024;
constexpr int DS_CAP = 16384;      // x + y entries an owner holds (128 KB)
constexpr int DS_OWN = 2048;       // buckets an owner can own

struct DsRec {
  double A, B;   // exclusive prefix over all buckets left of this one (fp64)
  float W, Z;    // this bucket's sums (rounded)
};

struct __align__(16) DsShared {
  float2 buf[DS_CAP];          // owner: x entries [0, Sx) then y entries [Sx, Sx + Sy), bucket order
  unsigned hxy[NB];            // local counters -> scatter cursors (x: low 16 bits, y: high 16 bits)
  unsigned oxy[DS_OWN + 1];    // owner: bucket starts (x | y << 16), y relative to Sx
  DsRec rec[DS_OWN];
  int2 gtab[NG];
  int gx[NG];
  int gxy[NG];
  int bnd[17];                 // bucket boundaries of the C owners
  int wbuf[34];
  int tot_i[4];
  double tot_d[4];
  double wsd[3][DS_T / 32];
  int ovf;
};

__device__ __forceinline__ int owner_of(int b, const int* bnd, int C) {
  int r = 0;
#pragma unroll
  for (int step = 8; step >= 1; step >>= 1)
    if (r + step < C && b >= bnd[r + step]) r += step;
  return r;
}

template <int C>
__global__ void __launch_bounds__(DS_T, 1) k_sortsum_dsm(SortArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  DsShared& S = *reinterpret_cast<DsShared*>(smraw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int slot = blockIdx.x / C, nslots = gridDim.x / C;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int W = DS_T / 32;
  const int64_t N = a.zv.N, M = a.zv.M;
  const int64_t x0 = N * rank / C, x1 = N * (rank + 1) / C;
  const int64_t y0 = M * rank / C, y1 = M * (rank + 1) / C;
  constexpr int U = 8;

  long long tph[10];
  int nph = 0;
#define PHASE() do { if (a.dbg && tid == 0 && p == slot) tph[nph++] = clock64(); } while (0)
  for (int p = slot; p < a.np; p += nslots) {
    PHASE();
    const float* zx = a.zv.zx + p * a.zv.ldx;
    const float* zy = a.zv.zy + p * a.zv.ldy;
    const float zmin = key2f_dev(a.mm[p * 4 + 0]), zmax = key2f_dev(a.mm[p * 4 + 1]);
    const float range = zmax - zmin;
    const float gscale = (range > 0.f) ? static_cast<float>(NG) / range : 0.f;
    if (rank == 0 && tid == 0) { a.bpar[p * 2 + 0] = zmin; a.bpar[p * 2 + 1] = gscale; }

    // ---- P0: granule histograms of my 1/C share -> bucket map + ownership (identical in every rank)
    for (int b = tid; b < NB; b += DS_T) S.hxy[b] = 0u;
    for (int g = tid; g < NG; g += DS_T) { S.gx[g] = 0; S.gxy[g] = 0; }
    if (tid == 0) S.ovf = 0;
    __syncthreads();
    for (int64_t base = x0; base < x1; base += U * DS_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * DS_T < x1) atomicAdd(&S.gx[gran_of(zz[k], zmin, gscale)], 1);
    }
    for (int64_t base = y0; base < y1; base += U * DS_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * DS_T < y1) atomicAdd(&S.gxy[gran_of(zz[k], zmin, gscale)], 1);
    }
    __syncthreads();
    for (int g = tid; g < NG; g += DS_T) S.gxy[g] += S.gx[g];
    cluster.sync();
    {
      __shared__ int gtx[NG], gtxy[NG];
      for (int g = tid; g < NG; g += DS_T) { gtx[g] = 0; gtxy[g] = 0; }
      __syncthreads();
      for (int e = tid; e < NG * C; e += DS_T) {   // all (granule, rank) remote reads in flight at once
        const int g = e % NG, r = e / NG;
        const DsShared* R = cluster.map_shared_rank(&S, r);
        const int vx = R->gx[g], vxy = R->gxy[g];
        atomicAdd(&gtx[g], vx);
        atomicAdd(&gtxy[g], vxy);
      }
      __syncthreads();
      if (wid == 0) {
        constexpr int PG = NG / 32;
        long long cx = 0, cxy = 0;
        for (int q = 0; q < PG; ++q) { cx += gtx[lane * PG + q]; cxy += gtxy[lane * PG + q]; }
        const long long ix = warp_incl_scan(cx), ixy = warp_incl_scan(cxy);
        const long long total = __shfl_sync(0xffffffffu, ixy, 31);
        long long cum = ix - cx, run = ixy - cxy;
        int prev = (N > 0) ? static_cast<int>((cum * NB) / N) : 0;
        for (int q = 0; q < PG; ++q) {
          const int g = lane * PG + q;
          cum += gtx[g];
          const int next = (N > 0) ? static_cast<int>((cum * NB) / N) : NB;
          S.gtab[g] = make_int2(prev, next - prev);
          prev = next;
          const long long before = run;
          run += gtxy[g];
          for (int r = 1; r < C; ++r)
            if (before * C < total * r && run * C >= total * r) S.wbuf[r] = g + 1;
        }
        if (lane == 0) {
          S.wbuf[0] = 0;
          S.wbuf[C] = NG;
          if (total == 0)
            for (int r = 1; r < C; ++r) S.wbuf[r] = NG;
        }
      }
      __syncthreads();
      if (tid <= C) S.bnd[tid] = (S.wbuf[tid] < NG) ? S.gtab[S.wbuf[tid]].x : NB;
      __syncthreads();
    }
    const int lo = S.bnd[rank], hi = S.bnd[rank + 1], nown = hi - lo;

    PHASE();
    // ---- P1: packed local counting
    for (int64_t base = x0; base < x1; base += U * DS_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * DS_T < x1) atomicAdd(&S.hxy[bin_of(zz[k], zmin, gscale, S.gtab)], 1u);
    }
    for (int64_t base = y0; base < y1; base += U * DS_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * DS_T < y1) atomicAdd(&S.hxy[bin_of(zz[k], zmin, gscale, S.gtab)], 0x10000u);
    }
    cluster.sync();

    PHASE();
    // ---- P2: owner totals, scans, capacity check, cursors into every rank
    int* tx = reinterpret_cast<int*>(S.rec);   // scratch: [DS_OWN] x totals, [DS_OWN] y totals
    int* ty = tx + DS_OWN;
    const bool own_ok = nown <= DS_OWN;
    if (own_ok) {
      for (int j = tid; j < nown; j += DS_T) { tx[j] = 0; ty[j] = 0; }
      __syncthreads();
      for (int e = tid; e < nown * C; e += DS_T) {   // (bucket, rank) pairs: independent remote reads
        const int j = e % nown, r = e / nown;
        const unsigned v = cluster.map_shared_rank(&S, r)->hxy[lo + j];
        if (v & 0xffffu) atomicAdd(&tx[j], static_cast<int>(v & 0xffffu));
        if (v >> 16) atomicAdd(&ty[j], static_cast<int>(v >> 16));
      }
    }
    __syncthreads();
    int Sx = 0, Sy = 0;
    if (own_ok) {
      Sx = block_scan_int(tx, nown, S.wbuf);
      Sy = block_scan_int(ty, nown, S.wbuf);
    }
    if (tid == 0) S.ovf = (!own_ok || Sx + Sy > DS_CAP) ? 1 : 0;
    cluster.sync();
    int any_ovf = 0;
    {
      int f = 0;
      if (lane < C) f = cluster.map_shared_rank(&S, lane)->ovf;
      any_ovf = __any_sync(0xffffffffu, f != 0);
    }
    if (any_ovf) {
      if (rank == 0 && tid == 0) a.ovf[p] = 1;
      cluster.sync();   // nobody still reads this slice's shared state
      continue;
    }
    // C consecutive lanes handle one bucket: lane r reads rank r's counters, a segmented shuffle scan over
    // the C lanes gives each rank's cursor base, lane r writes it back into rank r (all remote ops parallel)
    for (int e0 = 0; e0 < nown * C; e0 += DS_T) {
      const int e = e0 + tid;
      const bool act = e < nown * C;
      const int j = e / C, r = e % C;
      unsigned v = 0;
      if (act) v = cluster.map_shared_rank(&S, r)->hxy[lo + j];
      unsigned cx = v & 0xffffu, cy = v >> 16;
#pragma unroll
      for (int o = 1; o < C; o <<= 1) {   // inclusive scan within groups of C lanes (C divides 32)
        const unsigned nx = __shfl_up_sync(0xffffffffu, cx, o), ny = __shfl_up_sync(0xffffffffu, cy, o);
        if ((lane % C) >= o) { cx += nx; cy += ny; }
      }
      if (act) {
        const unsigned bx = static_cast<unsigned>(tx[j]) + cx - (v & 0xffffu);
        const unsigned by = static_cast<unsigned>(Sx + ty[j]) + cy - (v >> 16);
        cluster.map_shared_rank(&S, r)->hxy[lo + j] = bx | (by << 16);
        if (r == 0) S.oxy[j] = static_cast<unsigned>(tx[j]) | (static_cast<unsigned>(ty[j]) << 16);
      }
    }
    if (tid == 0) S.oxy[nown] = static_cast<unsigned>(Sx) | (static_cast<unsigned>(Sy) << 16);
    cluster.sync();

    PHASE();
    // ---- P3: scatter my share into the owners' shared memory (DSMEM stores)
    for (int64_t base = x0; base < x1; base += U * DS_T) {
      float zz[U], ww[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < x1) ? __ldg(zx + i) : 0.f;
        ww[k] = (i < x1) ? __ldg(a.w + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (base + tid + k * DS_T < x1) {
          const int b = bin_of(zz[k], zmin, gscale, S.gtab);
          const unsigned pos = atomicAdd(&S.hxy[b], 1u) & 0xffffu;
          cluster.map_shared_rank(&S, owner_of(b, S.bnd, C))->buf[pos] = make_float2(zz[k], ww[k]);
        }
    }
    for (int64_t base = y0; base < y1; base += U * DS_T) {
      float zz[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        zz[k] = (i < y1) ? __ldg(zy + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + tid + k * DS_T;
        if (i < y1) {
          const int b = bin_of(zz[k], zmin, gscale, S.gtab);
          const unsigned pos = atomicAdd(&S.hxy[b], 0x10000u) >> 16;
          cluster.map_shared_rank(&S, owner_of(b, S.bnd, C))->buf[pos] =
              make_float2(zz[k], __int_as_float(static_cast<int>(i)));
        }
      }
    }
    cluster.sync();

    PHASE();
    // ---- P4/P5: owner bucket sums (fp64, from shared memory), exclusive scan with cross-rank offsets
    const int per = (nown + DS_T - 1) / DS_T;
    const int j0 = min(nown, tid * per), j1 = min(nown, j0 + per);
    double lA = 0.0, lB = 0.0, lC = 0.0;
    for (int j = j0; j < j1; ++j) {
      const int xs0 = S.oxy[j] & 0xffff, xs1 = S.oxy[j + 1] & 0xffff;
      double Wb = 0.0, Zb = 0.0, Cb = 0.0;
      for (int i = xs0; i < xs1; ++i) {
        const float2 q = S.buf[i];
        const double wz = static_cast<double>(q.y) * q.x;
        Wb += q.y;
        Zb += wz;
        Cb += wz * q.x;
      }
      S.rec[j].W = static_cast<float>(Wb);   // rec[j].W / .Z overlap the tx/ty scratch only for j < DS_OWN/..:
      S.rec[j].Z = static_cast<float>(Zb);   // tx/ty are dead after P2 (their values live in oxy)
      S.rec[j].A = Wb;                       // temporarily the bucket sums (fp64)
      S.rec[j].B = Zb;
      lA += Wb;
      lB += Zb;
      lC += Cb;
    }
    {
      const double iA = warp_incl_scan(lA), iB = warp_incl_scan(lB);
      const double sC = warp_sum(lC);
      if (lane == 31) { S.wsd[0][wid] = iA; S.wsd[1][wid] = iB; }
      if (lane == 0) S.wsd[2][wid] = sC;
      __syncthreads();
      if (wid == 0) {
        const double va = S.wsd[0][lane], vb = S.wsd[1][lane], vc = S.wsd[2][lane];
        const double ia = warp_incl_scan(va), ib = warp_incl_scan(vb), sc = warp_sum(vc);
        S.wsd[0][lane] = ia - va;
        S.wsd[1][lane] = ib - vb;
        if (lane == 31) { S.tot_d[0] = ia; S.tot_d[1] = ib; }
        if (lane == 0) S.tot_d[2] = sc;
      }
      cluster.sync();
      __shared__ double xt[5];
      if (wid == 0) {   // lane r reads rank r's partial totals (parallel remote loads), warp reductions
        double ta = 0, tb = 0, tc = 0;
        if (lane < C) {
          const DsShared* R = cluster.map_shared_rank(&S, lane);
          ta = R->tot_d[0]; tb = R->tot_d[1]; tc = R->tot_d[2];
        }
        const double pa = warp_sum(lane < rank ? ta : 0.0), pb = warp_sum(lane < rank ? tb : 0.0);
        ta = warp_sum(ta); tb = warp_sum(tb); tc = warp_sum(tc);
        if (lane == 0) { xt[0] = ta; xt[1] = tb; xt[2] = tc; xt[3] = pa; xt[4] = pb; }
      }
      __syncthreads();
      const double TA = xt[0], TB = xt[1], TC = xt[2], PA = xt[3], PB = xt[4];
      if (rank == 0 && tid == 0) a.tot[p] = SliceTot{TA, TB, TC, 0.0};
      double rA = PA + S.wsd[0][wid] + iA - lA, rB = PB + S.wsd[1][wid] + iB - lB;
      for (int j = j0; j < j1; ++j) {
        const double Wb = S.rec[j].A, Zb = S.rec[j].B;
        S.rec[j].A = rA;
        S.rec[j].B = rB;
        rA += Wb;
        rB += Zb;
      }
      __syncthreads();

      PHASE();
      // ---- P6: my targets in bucket order, everything from shared memory
      const int Sy0 = Sx;
      for (int e = tid; e < Sy; e += DS_T) {
        const float2 y = S.buf[Sy0 + e];
        const float z = y.x;
        const int64_t m = __float_as_int(y.y);
        const int jb = bin_of(z, zmin, gscale, S.gtab) - lo;
        const DsRec R = S.rec[jb];
        const int xs0 = S.oxy[jb] & 0xffff, xs1 = S.oxy[jb + 1] & 0xffff;
        float s0 = 0.f, s1 = 0.f;
        int i = xs0;
        for (; i + 2 <= xs1; i += 2) {
          const float2 q0 = S.buf[i], q1 = S.buf[i + 1];
          s0 = fmaf(q0.y, fabsf(q0.x - z), s0);
          s1 = fmaf(q1.y, fabsf(q1.x - z), s1);
        }
        if (i < xs1) {
          const float2 q = S.buf[i];
          s0 = fmaf(q.y, fabsf(q.x - z), s0);
        }
        const double zd = z;
        const double Ahi = TA - R.A - R.W, Bhi = TB - R.B - R.Z;
        const double t = -a.coef * ((zd * R.A - R.B) + (Bhi - zd * Ahi) + static_cast<double>(s0 + s1));
        if (a.s64) atomicAdd(a.s64 + m, t);
        if (a.per_slice_out) a.per_slice_out[static_cast<int64_t>(p) * M + m] = static_cast<float>(t);
      }
    }
    PHASE();
    cluster.sync();   // shared state is reused by the next slice
  }
  if (a.dbg && tid == 0)
    for (int k = 0; k + 1 < nph; ++k) a.dbg[static_cast<int64_t>(blockIdx.x) * 8 + k] = tph[k + 1] - tph[k];
#undef PHASE
}

}  // namespace

int sortpath_buckets() { return NB; }

int sortpath_slots(int np) {
  static int nclusters = 0;
  if (nclusters == 0) {
    cudaFuncSetAttribute(k_sortsum, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Shared)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(SP_C * 64);
    cfg.blockDim = dim3(SP_T);
    cfg.dynamicSmemBytes = sizeof(Shared);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = SP_C;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_sortsum, &cfg) != cudaSuccess || n <= 0) n = 148 / SP_C;
    nclusters = n;
  }
  return np < nclusters ? np : nclusters;
}

namespace {
template <int C>
int dsm_clusters() {
  static int n = -1;
  if (n < 0) {
    cudaFuncSetAttribute(k_sortsum_dsm<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(DsShared)));
    if (C > 8) cudaFuncSetAttribute(k_sortsum_dsm<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C * 16);
    cfg.blockDim = dim3(DS_T);
    cfg.dynamicSmemBytes = sizeof(DsShared);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = C;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int k = 0;
    if (cudaOccupancyMaxActiveClusters(&k, k_sortsum_dsm<C>, &cfg) != cudaSuccess) k = 0;
    cudaGetLastError();
    n = k;
  }
  return n;
}

template <int C>
cudaError_t launch_dsm(const SortArgs& a, int nclusters, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(C * nclusters));
  cfg.blockDim = dim3(DS_T);
  cfg.dynamicSmemBytes = sizeof(DsShared);
  cfg.stream = st;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = C;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_sortsum_dsm<C>, a);
}
}  // namespace

cudaError_t launch_sortpath(const SortArgs& a0, int slots, cudaStream_t st) {
  SortArgs a = a0;
  const int64_t L = a.zv.N + a.zv.M;
  // DSMEM-resident path when an evenly balanced owner holds <= 80% of its capacity
  int C = 0;
  if (L * 10 <= static_cast<int64_t>(DS_CAP) * 8 * 8) C = 8;
  else if (L * 10 <= static_cast<int64_t>(DS_CAP) * 16 * 8) C = 16;
  // measured on B200 (cfg2): the 4-CTA global-scratch kernel (1.44 ms) beats the DSMEM-resident one (2.0-2.3 ms,
  // DSMEM stores are transaction-bound like scattered global stores and only 8 16-CTA clusters fit); opt-in
  if (!std::getenv("SKS_SORT_DSM")) C = 0;
  if (C) {
    const int ncl = (C == 8) ? dsm_clusters<8>() : dsm_clusters<16>();
    if (ncl > 0) {
      cudaError_t e = cudaMemsetAsync(a.ovf, 0, sizeof(int) * a.np, st);
      if (e != cudaSuccess) return e;
      const int n = a.np < ncl ? a.np : ncl;
      e = (C == 8) ? launch_dsm<8>(a, n, st) : launch_dsm<16>(a, n, st);
      if (e != cudaSuccess) return e;
      a.only_flagged = 1;   // the global kernel redoes only the slices the DSMEM kernel flagged
    }
  }
  k_sortsum<<<slots * SP_C, SP_T, sizeof(Shared), st>>>(a);
  return cudaGetLastError();
}

}  // namespace sks
