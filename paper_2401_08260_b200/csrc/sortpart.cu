// sortpart.cu -- the sort path (rows a3 + a4) as an owner-partitioned counting sort.
//
// Sec. 3.2 / Alg. 2 computes, exactly,
//     t_m = -c sum_n w_n |x_n - y_m|                               (c = c_d, or alpha c_d, Laplacian)
// by sorting the projections and taking prefix sums of w and w x.  Any monotone non-decreasing key map
// k(z) gives the same identity: for a target z,
//     sum_n w_n |x_n - z| = [z A_lo - B_lo] + [B_hi - z A_hi] + sum_{x: k(x) = k(z)} w |x - z|
// where (A, B)_{lo/hi} = (sum w, sum w x) over the x with k(x) < k(z) (which are <= z) / k(x) > k(z)
// (which are >= z); ties contribute |x - z| = 0 on either side.
//
// B200 design (measured, scratch/ubench_scatter.cu): a scattered 4-8 byte global or DSMEM access costs
// 1-3 SM cycles per element, a random local shared-memory access 0.2.  So every random access of the
// method is kept in the local shared memory of one CTA, and data moves between CTAs only in coalesced runs:
//   S0 k_sp_hist   per chunk: histogram of the x and y projections over NH equal bins of [xmin, xmax] into the
//                  chunk's own slot (no global atomics); the last chunk of a slice sums them
//                  (+ slice totals sum w, sum w x, sum w x^2 in fp64 for the Laplacian moment term)
//   S1 k_sp_plan   per slice: bins -> G owners balanced by x count (owner = contiguous bin range, so the
//                  key k = (owner, fine bucket) stays monotone); region offsets of every owner
//   S2 k_sp_part   per chunk: local counting sort of the chunk by owner in shared memory, runs appended to
//                  the owners' mailbox regions (x: (z, w); y: z) with coalesced stores; y positions recorded;
//                  per-owner fp64 sums of w and w x
//   S3 k_sp_owner  per (owner, slice): the owner's x into NBF fine buckets in shared memory (counting sort),
//                  fp64 exclusive bucket prefix sums, then every y of the owner evaluated from shared memory
//                  only; t (fp32) written at the y's mailbox position (coalesced)
//   S4 k_sp_gather per (target chunk, slice group): the other owners' contribution table from the owners'
//                  fp64 totals (in shared memory), t gathered back to target order through the recorded
//                  positions, accumulated over slices in fp64 registers, one coalesced atomic per target
// An owner whose x exceed the shared-memory capacity (degenerate data: one bin holding > SP_CAP points) is
// processed in several passes over subsets of its x (the identity is additive over the sources).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>

#include "kernels.h"

namespace sks {

namespace {

constexpr int S0_T = 512;      // histogram threads
// owner kernel shape (x capacity, fine buckets, CTAs per SM, threads).  Measured on B200, cfg2 sp_owner (one
// stream): {4096,1024,3,512} 358 us (kept), {8192,2048,2,512} 438, {4096,1024,4,256} 389, {2048,1024,4,512} 465,
// {4096,1024,2,512} 401; finer buckets {4096,2048,3,512} 418.  At d = 100, P = 1000, N = 1e6 / 1e7 (ms): kept
// 34.5 / 489, the others 35.5-40.2 / 485-588.
constexpr int SP_CAP = 4096, SP_NBF = 1024, SP_MINB = 3, SP_NT = 512;
static_assert(SP_CAP < 65536, "bucket bounds packed as 16-bit pairs (OwnerShared::se)");
constexpr int S4_T = 256, S4_PER = 4, S4_CH = S4_T * S4_PER;    // gather
constexpr int S4_SG = 8;   // slices per gather thread (measured 4 / 8 / 16 / 32: 8 best; also on the global-table
                           // path at N = 1e7, P = 1000: 8 / 16 / 32 -> 489 / 494 / 507 ms, scratch/gsg.sh)
constexpr int kSmemDabMax = 128;   // owners per slice up to which the gather builds the other-owner table itself
constexpr int S0_CH = 32768;   // histogram: elements per CTA (measured 8192 / 16384 / 32768: the largest best)

__device__ __forceinline__ float key2f_sp(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// L2-cached loads (no L1 allocation); plain loads so that the compiler can keep many in flight
__device__ __forceinline__ float ldg_cg(const float* p) {
  float v;
  asm("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldg_cg2(const float2* p) {
  float2 v;
  asm("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// bin coordinate u = (z - xmin) * hscale with explicitly rounded fp32 ops: monotone non-decreasing in z
// u = z hscale + uoff (uoff = -xmin hscale), one correctly rounded FMA: monotone non-decreasing in z
__device__ __forceinline__ float ucoord(float z, float uoff, float hscale) { return fmaf(z, hscale, uoff); }
// floor(v) clamped to [0, n): monotone (saturating truncation; equals floor for v >= 0); NaN -> 0
__device__ __forceinline__ int clamp_floor(float v, int n) { return min(max(__float2int_rz(v), 0), n - 1); }
// fine bucket inside an owner: monotone in u (hence in z)
template <int NBF>
__device__ __forceinline__ int fine_of(float u, float blo, float fmul) {
  return clamp_floor(fmaf(u, fmul, -blo * fmul), NBF);
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan_sp(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum_sp(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// exclusive scan of one value per thread over the CTA (NT threads); returns the exclusive prefix, *total
// gets the CTA total.  wbuf: >= NT/32 + 1 elements of shared memory.
template <int NT, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* wbuf, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  const T inc = warp_incl_scan_sp(v);
  if (lane == 31) wbuf[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const T x = (lane < NW) ? wbuf[lane] : T(0);
    const T xi = warp_incl_scan_sp(x);
    if (lane < NW) wbuf[lane] = xi - x;
    if (lane == NW - 1) wbuf[NW] = xi;
  }
  __syncthreads();
  const T r = wbuf[wid] + inc - v;
  *total = wbuf[NW];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------------------- S0 + S1
// Histogram of one chunk (x or y part of a slice); the last CTA of a slice to finish builds the slice's plan
// (ticket counter per slice): owner of bin b = floor(cx[b] G / Nx) with cx the exclusive prefix x count, so
// the owners are contiguous bin ranges (monotone) holding <= Nx/G + (largest bin) x each.
__global__ void __launch_bounds__(S0_T) k_sp_hist(ZView zv, const unsigned* __restrict__ mm, int NH, int G,
                                                  int ncx, int nchunks, int chx, int chy, int NBF, int* __restrict__ H,
                                                  int* __restrict__ done, uint16_t* __restrict__ om,
                                                  SpOwner* __restrict__ own, int* __restrict__ base, int base_par) {
  extern __shared__ int hs[];   // [NH] histogram; in the plan: cx[NH + 1], cy[NH + 1], blo[G + 1]
  __shared__ int wbuf[S0_T / 32 + 1];
  __shared__ int last;
  const int p = blockIdx.y, tid = threadIdx.x;
  const bool isx = static_cast<int>(blockIdx.x) < ncx;
  const int c = isx ? blockIdx.x : blockIdx.x - ncx;
  const int n = static_cast<int>(isx ? zv.N : zv.M);
  const float* z = isx ? zv.zx + p * zv.ldx : zv.zy + p * zv.ldy;
  const int ch = isx ? chx : chy;
  const int i0 = c * ch, i1 = min(n, i0 + ch);
  const float xmin = key2f_sp(mm[p * 4 + 0]), xmax = key2f_sp(mm[p * 4 + 1]);
  const float hscale = (xmax > xmin) ? static_cast<float>(NH) / (xmax - xmin) : 0.f;
  const float uoff = -xmin * hscale;
  for (int b = tid; b < NH; b += S0_T) hs[b] = 0;
  __syncthreads();
  // 16-byte loads on the aligned body of the chunk, scalar head / tail
  const int mis = static_cast<int>((reinterpret_cast<uintptr_t>(z + i0) >> 2) & 3);
  const int ia = min(i1, i0 + ((4 - mis) & 3)), nv = (i1 - ia) >> 2, ib = ia + 4 * nv;
  if (tid < ia - i0) atomicAdd(&hs[clamp_floor(ucoord(__ldg(z + i0 + tid), uoff, hscale), NH)], 1);
  if (tid < i1 - ib) atomicAdd(&hs[clamp_floor(ucoord(__ldg(z + ib + tid), uoff, hscale), NH)], 1);
  const float4* z4 = reinterpret_cast<const float4*>(z + ia);
  constexpr int U = 4;
  for (int base = 0; base < nv; base += U * S0_T) {
    float4 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int v = base + tid + k * S0_T;
      q[k] = (v < nv) ? __ldg(z4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (base + tid + k * S0_T < nv) {
        atomicAdd(&hs[clamp_floor(ucoord(q[k].x, uoff, hscale), NH)], 1);
        atomicAdd(&hs[clamp_floor(ucoord(q[k].y, uoff, hscale), NH)], 1);
        atomicAdd(&hs[clamp_floor(ucoord(q[k].z, uoff, hscale), NH)], 1);
        atomicAdd(&hs[clamp_floor(ucoord(q[k].w, uoff, hscale), NH)], 1);
      }
  }
  __syncthreads();
  // the chunk's histogram into its own slot (plain coalesced stores; the plan sums the chunks)
  int* Hp = H + (static_cast<int64_t>(p) * nchunks + blockIdx.x) * NH;
  for (int b = tid; b < NH; b += S0_T) __stcg(Hp + b, hs[b]);
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(done + p, 1) == nchunks - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // ---- plan of slice p (this CTA saw every chunk's histogram)
  int* cx = hs;
  int* cy = cx + NH + 1;
  int* blo = cy + NH + 1;
  const int* hp = H + static_cast<int64_t>(p) * nchunks * NH;
  // per bin: x and y counts summed over the chunks (into cx / cy, then scanned in place)
  for (int b = tid; b < NH; b += S0_T) {
    int sx = 0, sy = 0;
    for (int q = 0; q < ncx; ++q) sx += __ldcg(hp + static_cast<int64_t>(q) * NH + b);
    for (int q = ncx; q < nchunks; ++q) sy += __ldcg(hp + static_cast<int64_t>(q) * NH + b);
    cx[b] = sx;
    cy[b] = sy;
  }
  __syncthreads();
  const int per = (NH + S0_T - 1) / S0_T;
  const int b0 = min(NH, tid * per), b1 = min(NH, b0 + per);
  int lx = 0, ly = 0;
  for (int b = b0; b < b1; ++b) { lx += cx[b]; ly += cy[b]; }
  int tx, ty;
  int rx = block_excl_scan<S0_T>(lx, wbuf, &tx);
  int ry = block_excl_scan<S0_T>(ly, wbuf, &ty);
  for (int b = b0; b < b1; ++b) {
    const int vx = cx[b], vy = cy[b];
    cx[b] = rx; cy[b] = ry;
    rx += vx; ry += vy;
  }
  if (tid == 0) { cx[NH] = tx; cy[NH] = ty; }
  for (int o = tid; o <= G; o += S0_T) blo[o] = (o == 0) ? 0 : NH;
  __syncthreads();
  const int64_t Nx = (tx > 0) ? tx : 1;
  for (int b = tid; b < NH; b += S0_T) {
    const int oo = min(G - 1, static_cast<int>((static_cast<int64_t>(cx[b]) * G) / Nx));
    om[static_cast<int64_t>(p) * NH + b] = static_cast<uint16_t>(oo);
    const int prev = (b == 0) ? -1 : min(G - 1, static_cast<int>((static_cast<int64_t>(cx[b - 1]) * G) / Nx));
    for (int q = prev + 1; q <= oo; ++q) blo[q] = b;   // owners prev+1 .. oo start at bin b (skipped ones empty)
  }
  __syncthreads();
  for (int o = tid; o < G; o += S0_T) {
    const int lo = blo[o];
    const int hi = (o + 1 < G) ? blo[o + 1] : NH;
    SpOwner r;
    r.xoff = cx[lo];
    r.xcnt = cx[hi] - cx[lo];
    r.yoff = cy[lo];
    r.ycnt = cy[hi] - cy[lo];
    r.blo = static_cast<float>(lo);
    r.fmul = (hi > lo) ? static_cast<float>(NBF) / static_cast<float>(hi - lo) : 0.f;
    r.pad0 = r.pad1 = 0;
    own[static_cast<int64_t>(p) * G + o] = r;
  }
  if (base == nullptr) return;
  // many owners: the first mailbox slot of every (chunk, owner) -- the owner's region start plus its counts in
  // the earlier chunks of the same part -- so that the partition needs no run reservations (k_sp_part_big)
  __syncthreads();
  if (base_par) {   // all chunks at once: cnt[nchunks][G] fits in shared memory
    int* cnt = blo + G + 1;
    for (int e = tid; e < nchunks * G; e += S0_T) cnt[e] = 0;
    __syncthreads();
    for (int b = tid; b < NH; b += S0_T) {
      const int oo = min(G - 1, static_cast<int>((static_cast<int64_t>(cx[b]) * G) / Nx));
      for (int q = 0; q < nchunks; ++q) {
        const int v = __ldcg(hp + static_cast<int64_t>(q) * NH + b);
        if (v) atomicAdd(&cnt[q * G + oo], v);
      }
    }
    __syncthreads();
    for (int o = tid; o < G; o += S0_T) {
      const int lo = blo[o];
      int rx = cx[lo], ry = cy[lo];
      int* bp = base + static_cast<int64_t>(p) * nchunks * G + o;
      for (int q = 0; q < ncx; ++q) { bp[q * G] = rx; rx += cnt[q * G + o]; }
      for (int q = ncx; q < nchunks; ++q) { bp[q * G] = ry; ry += cnt[q * G + o]; }
    }
    return;
  }
  // else one chunk at a time (shared memory O(G))
  int* cnt = blo + G + 1;   // [G] the current chunk's count per owner
  int* runx = cnt + G;      // [G] running x slot per owner
  int* runy = runx + G;     // [G] running y slot per owner
  for (int o = tid; o < G; o += S0_T) { runx[o] = cx[blo[o]]; runy[o] = cy[blo[o]]; }
  __syncthreads();
  int* bown = cy;           // cy is spent: the owner of each bin (one division per bin, not one per chunk)
  for (int b = tid; b < NH; b += S0_T) bown[b] = min(G - 1, static_cast<int>((static_cast<int64_t>(cx[b]) * G) / Nx));
  for (int q = 0; q < nchunks; ++q) {
    for (int o = tid; o < G; o += S0_T) cnt[o] = 0;
    __syncthreads();
    for (int b = tid; b < NH; b += S0_T) {
      const int v = __ldcg(hp + static_cast<int64_t>(q) * NH + b);
      if (v) atomicAdd(&cnt[bown[b]], v);
    }
    __syncthreads();
    int* bp = base + (static_cast<int64_t>(p) * nchunks + q) * G;
    int* run = q < ncx ? runx : runy;
    for (int o = tid; o < G; o += S0_T) { bp[o] = run[o]; run[o] += cnt[o]; }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------- S2
// Warp-level partition by owner, no block barriers: a warp takes 256 consecutive elements of a slice part
// (8 rounds of 32), ranks them per owner with shared-memory counters private to the warp, reserves one run
// per (warp, owner) in the owner's mailbox region with one global atomic, and stores each element at
// region + run + rank (runs of ~256/G consecutive slots).  For y it also records, in target order, the
// mailbox slot (ypos) and the owner (yown).  No sums here: every owner sums its own x (k_sp_owner).
constexpr int S2W_T = 256, S2W_WARPS = S2W_T / 32, S2W_PER = 8, S2W_WCH = 32 * S2W_PER;

// one round of one warp: 256 consecutive elements [e0, e0 + 256) of a slice part (FULL: all in range)
template <bool IsX, bool FULL>
__device__ __forceinline__ void part_round(int e0, int n, const float* __restrict__ z, const float* __restrict__ w,
                                           float uoff, float hscale, int NH, int G, const uint16_t* om, const int* ooff,
                                           int* cw, int* curp, float2* __restrict__ xdst, float* __restrict__ ydst,
                                           int* __restrict__ yp, uint16_t* __restrict__ yo) {
  const int lane = threadIdx.x & 31;
  for (int o = lane; o < G; o += 32) cw[o] = 0;
  float zz[S2W_PER], ww[S2W_PER];
#pragma unroll
  for (int k = 0; k < S2W_PER; ++k) {
    const int i = e0 + 32 * k + lane;
    zz[k] = (FULL || i < n) ? __ldg(z + i) : 0.f;
    if (IsX) ww[k] = (FULL || i < n) ? __ldg(w + i) : 0.f;
  }
  __syncwarp();
  int ow[S2W_PER], rk[S2W_PER];
#pragma unroll
  for (int k = 0; k < S2W_PER; ++k) {
    ow[k] = -1;
    if (FULL || e0 + 32 * k + lane < n) {
      ow[k] = om[clamp_floor(ucoord(zz[k], uoff, hscale), NH)];
      rk[k] = atomicAdd(&cw[ow[k]], 1);
    }
  }
  __syncwarp();
  for (int o = lane; o < G; o += 32) {   // one run per (warp, owner): counter -> absolute slot of the run
    const int c = cw[o];
    cw[o] = c ? ooff[o] + atomicAdd(curp + o, c) : 0;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < S2W_PER; ++k) {
    if (!FULL && ow[k] < 0) continue;
    const int dst = cw[ow[k]] + rk[k];
    const int i = e0 + 32 * k + lane;
    SKS_CHECK(dst >= 0 && dst < n && ow[k] < G);
    if (IsX) {
      xdst[dst] = make_float2(zz[k], ww[k]);
    } else {
      ydst[dst] = zz[k];
      yp[i] = dst;
      yo[i] = static_cast<uint16_t>(ow[k]);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(S2W_T) k_sp_part(ZView zv, const float* __restrict__ w, const unsigned* __restrict__ mm,
                                                   int NH, int G, int ncx, int wpc, const uint16_t* __restrict__ om_g,
                                                   const SpOwner* __restrict__ own, int* __restrict__ cursor,
                                                   float2* __restrict__ Xmb, float* __restrict__ Ymb,
                                                   int* __restrict__ ypos, uint16_t* __restrict__ yown) {
  extern __shared__ __align__(16) unsigned char sh2[];
  int* ooff = reinterpret_cast<int*>(sh2);                              // [G] region start of each owner
  int* cntw = ooff + G;                                                 // [warps][G] per-warp counters / runs
  uint16_t* om = reinterpret_cast<uint16_t*>(ooff + ((1 + S2W_WARPS) * G + 3) / 4 * 4);   // [NH], 16-B aligned
  const int p = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool isx = static_cast<int>(blockIdx.x) < ncx;
  const int cb = isx ? blockIdx.x : blockIdx.x - ncx;
  const int n = static_cast<int>(isx ? zv.N : zv.M);
  const float* z = isx ? zv.zx + p * zv.ldx : zv.zy + p * zv.ldy;
  const float xmin = key2f_sp(mm[p * 4 + 0]), xmax = key2f_sp(mm[p * 4 + 1]);
  const float hscale = (xmax > xmin) ? static_cast<float>(NH) / (xmax - xmin) : 0.f;
  const float uoff = -xmin * hscale;
  {
    const uint4* src = reinterpret_cast<const uint4*>(om_g + static_cast<int64_t>(p) * NH);   // NH % 8 == 0
    uint4* dst = reinterpret_cast<uint4*>(om);
    for (int b = tid; b < NH / 8; b += S2W_T) dst[b] = __ldg(src + b);
    const SpOwner* ownp = own + static_cast<int64_t>(p) * G;
    for (int o = tid; o < G; o += S2W_T) ooff[o] = isx ? ownp[o].xoff : ownp[o].yoff;
  }
  __syncthreads();
  int* cw = cntw + wid * G;
  int* curp = cursor + static_cast<int64_t>(p) * 2 * G + (isx ? 0 : G);
  float2* xdst = Xmb + static_cast<int64_t>(p) * zv.N;
  float* ydst = Ymb + static_cast<int64_t>(p) * zv.M;
  for (int it = 0; it < wpc; ++it) {
    const int e0 = ((cb * wpc + it) * S2W_WARPS + wid) * S2W_WCH;   // this warp's 256 elements
    if (e0 >= n) break;   // warp-uniform
    const bool full = e0 + S2W_WCH <= n;   // warp-uniform: no per-element bounds in the common case
    if (isx) {
      if (full) part_round<true, true>(e0, n, z, w, uoff, hscale, NH, G, om, ooff, cw, curp, xdst, ydst, nullptr, nullptr);
      else part_round<true, false>(e0, n, z, w, uoff, hscale, NH, G, om, ooff, cw, curp, xdst, ydst, nullptr, nullptr);
    } else {
      int* yp = ypos + static_cast<int64_t>(p) * zv.M;
      uint16_t* yo = yown + static_cast<int64_t>(p) * zv.M;
      if (full) part_round<false, true>(e0, n, z, w, uoff, hscale, NH, G, om, ooff, cw, curp, xdst, ydst, yp, yo);
      else part_round<false, false>(e0, n, z, w, uoff, hscale, NH, G, om, ooff, cw, curp, xdst, ydst, yp, yo);
    }
  }
}

// Many owners (G > kSmemDabMax): one CTA per histogram chunk; the plan gave every (chunk, owner) its first mailbox
// slot, so no global atomics are needed (with the per-warp-round reservations above, a round of 256 elements over
// ~1000 owners costs about one global atomic per element).  The chunk is processed in sub-chunks of SB elements,
// each counting-sorted by owner in shared memory before it is written, so that an owner's elements of the
// sub-chunk leave as one contiguous run (the mailbox writes are otherwise 8-byte scatters over ~1000 regions).
template <int NT, int SB_PER>
__global__ void __launch_bounds__(NT) k_sp_part_big(ZView zv, const float* __restrict__ w, const unsigned* __restrict__ mm,
                                                      int NH, int G, int ncx, int nchunks, int chx, int chy,
                                                      const uint16_t* __restrict__ om_g, const int* __restrict__ base,
                                                      float2* __restrict__ Xmb, float* __restrict__ Ymb,
                                                      int* __restrict__ ypos, uint16_t* __restrict__ yown) {
  constexpr int SB = NT * SB_PER;   // elements per sub-chunk
  extern __shared__ __align__(16) unsigned char shb[];
  const int G4 = (G + 3) / 4 * 4;
  int* gnext = reinterpret_cast<int*>(shb);               // [G] next mailbox slot of each owner (this chunk)
  int* lcnt = gnext + G4;                                 // [G] sub-chunk counts, then exclusive starts
  float2* stg = reinterpret_cast<float2*>(lcnt + G4);     // [SB] sub-chunk elements in owner order
  uint16_t* sow = reinterpret_cast<uint16_t*>(stg + SB);  // [SB] owner of each staged element
  uint16_t* om = sow + SB;                                // [NH]
  __shared__ int wbuf[NT / 32 + 1];
  const int p = blockIdx.y, tid = threadIdx.x;
  const bool isx = static_cast<int>(blockIdx.x) < ncx;
  const int c = isx ? blockIdx.x : blockIdx.x - ncx;
  const int n = static_cast<int>(isx ? zv.N : zv.M);
  const int ch = isx ? chx : chy;
  const float* z = isx ? zv.zx + p * zv.ldx : zv.zy + p * zv.ldy;
  const float xmin = key2f_sp(mm[p * 4 + 0]), xmax = key2f_sp(mm[p * 4 + 1]);
  const float hscale = (xmax > xmin) ? static_cast<float>(NH) / (xmax - xmin) : 0.f;
  const float uoff = -xmin * hscale;
  {
    const uint4* src = reinterpret_cast<const uint4*>(om_g + static_cast<int64_t>(p) * NH);   // NH % 8 == 0
    uint4* dst = reinterpret_cast<uint4*>(om);
    for (int b = tid; b < NH / 8; b += NT) dst[b] = __ldg(src + b);
    const int* bp = base + (static_cast<int64_t>(p) * nchunks + blockIdx.x) * G;
    for (int o = tid; o < G; o += NT) gnext[o] = __ldg(bp + o);
  }
  const int i0 = c * ch, i1 = min(n, i0 + ch);
  float2* xdst = Xmb + static_cast<int64_t>(p) * zv.N;
  float* ydst = Ymb + static_cast<int64_t>(p) * zv.M;
  int* yp = ypos + static_cast<int64_t>(p) * zv.M;
  uint16_t* yo = yown + static_cast<int64_t>(p) * zv.M;
  for (int e0 = i0; e0 < i1; e0 += SB) {
    for (int o = tid; o < G; o += NT) lcnt[o] = 0;
    __syncthreads();
    float zz[SB_PER], ww[SB_PER];
    int ow[SB_PER], rk[SB_PER];
#pragma unroll
    for (int k = 0; k < SB_PER; ++k) {
      const int i = e0 + k * NT + tid;
      zz[k] = i < i1 ? __ldg(z + i) : 0.f;
      ww[k] = (isx && i < i1) ? __ldg(w + i) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < SB_PER; ++k) {
      ow[k] = -1;
      if (e0 + k * NT + tid < i1) {
        ow[k] = om[clamp_floor(ucoord(zz[k], uoff, hscale), NH)];
        rk[k] = atomicAdd(&lcnt[ow[k]], 1);
      }
    }
    __syncthreads();
    // exclusive starts of the owners in the sub-chunk (blocked: thread t scans owners [t * per, (t+1) * per))
    const int per = (G + NT - 1) / NT;
    const int o0 = min(G, tid * per), o1 = min(G, o0 + per);
    int loc = 0;
    for (int o = o0; o < o1; ++o) loc += lcnt[o];
    int tot;
    int run = block_excl_scan<NT>(loc, wbuf, &tot);
    for (int o = o0; o < o1; ++o) { const int v = lcnt[o]; lcnt[o] = run; run += v; }
    __syncthreads();
    // stage in owner order; y: positions / owners straight to target order
#pragma unroll
    for (int k = 0; k < SB_PER; ++k) {
      if (ow[k] < 0) continue;
      const int sidx = lcnt[ow[k]] + rk[k];
      stg[sidx] = make_float2(zz[k], ww[k]);
      sow[sidx] = static_cast<uint16_t>(ow[k]);
      if (!isx) {
        const int i = e0 + k * NT + tid;
        yp[i] = gnext[ow[k]] + rk[k];
        yo[i] = static_cast<uint16_t>(ow[k]);
      }
    }
    __syncthreads();
    // write out in owner order: consecutive staging slots of an owner -> consecutive mailbox slots
    for (int sidx = tid; sidx < tot; sidx += NT) {
      const int o = sow[sidx];
      const int dst = gnext[o] + (sidx - lcnt[o]);
      const float2 v = stg[sidx];
      if (isx) xdst[dst] = v;
      else ydst[dst] = v.x;
    }
    __syncthreads();
    // advance the owners' next slots by their sub-chunk counts (counts = next start - start)
    for (int o = o0; o < o1; ++o) gnext[o] += ((o + 1 < G) ? lcnt[o + 1] : tot) - lcnt[o];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------- S3
template <int SP_CAP, int SP_NBF, int NT>
struct __align__(16) OwnerShared {
  float2 xs[SP_CAP];          // the pass's x (z, w) in fine-bucket order
  double2 rec[SP_NBF + 1];    // exclusive prefix (sum w, sum w x) over the pass's buckets; [NBF] = pass totals
  int start[SP_NBF + 1];      // bucket b holds xs[start[b], start[b+1])
  unsigned se[SP_NBF];        // start[b] | start[b+1] << 16 in one 4-byte word for the lookups (SP_CAP <= 8192):
                              // a random 4-byte lookup costs fewer shared-memory wavefronts than an 8-byte one
  int wbuf[NT / 32 + 1];
  double2 dbuf[NT / 32 + 1];
};

__device__ __forceinline__ double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 operator-(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 shfl_up_d2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}

// exclusive block scan of a double2 per thread (NT threads)
template <int NT>
__device__ __forceinline__ double2 block_excl_scan_d2(double2 v, double2* wbuf, double2* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  double2 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double2 nb = shfl_up_d2(inc, o);
    if (lane >= o) inc = inc + nb;
  }
  if (lane == 31) wbuf[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const double2 x = (lane < NW) ? wbuf[lane] : make_double2(0.0, 0.0);
    double2 xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double2 nb = shfl_up_d2(xi, o);
      if (lane >= o) xi = xi + nb;
    }
    if (lane < NW) wbuf[lane] = xi - x;
    if (lane == NW - 1) wbuf[NW] = xi;
  }
  __syncthreads();
  const double2 r = wbuf[wid] + inc - v;
  *total = wbuf[NW];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int2 se_unpack(unsigned v) { return make_int2(static_cast<int>(v & 0xffffu), static_cast<int>(v >> 16)); }

template <int SP_CAP, int SP_NBF, int MINB, int S3_T>
__global__ void __launch_bounds__(S3_T, MINB) k_sp_owner(const SpOwner* __restrict__ own, double* __restrict__ otot,
                                                      const unsigned* __restrict__ mm, int NH, int G, int64_t N,
                                                      int64_t M, const float2* __restrict__ Xmb,
                                                      const float* __restrict__ Ymb, double coef, float* __restrict__ R,
                                                      int det) {
  extern __shared__ __align__(16) unsigned char sh3[];
  constexpr int S3_PER = SP_CAP / S3_T;
  OwnerShared<SP_CAP, SP_NBF, S3_T>& S = *reinterpret_cast<OwnerShared<SP_CAP, SP_NBF, S3_T>*>(sh3);
  const int o = blockIdx.x, p = blockIdx.y, tid = threadIdx.x;
  const SpOwner r = own[static_cast<int64_t>(p) * G + o];
  // every owner publishes its x totals (sum w, sum w z, sum w z^2; fp64) for the other owners' targets
  // (k_sp_gather's other-owner table), so an owner without targets still sums its x
  __shared__ double own_tot[3];
  __shared__ double wvc[S3_T / 32];   // per-warp sum w z^2 of the pass (shared fp64 atomics are CAS loops)
  if (tid < 3) own_tot[tid] = 0.0;
  const float xmin = key2f_sp(mm[p * 4 + 0]), xmax = key2f_sp(mm[p * 4 + 1]);
  const float hscale = (xmax > xmin) ? static_cast<float>(NH) / (xmax - xmin) : 0.f;
  const float uoff = -xmin * hscale;
  const float2* xsrc = Xmb + static_cast<int64_t>(p) * N + r.xoff;
  const float* ysrc = Ymb + static_cast<int64_t>(p) * M + r.yoff;
  float* rdst = R + static_cast<int64_t>(p) * M + r.yoff;
  const int npass = (r.xcnt + SP_CAP - 1) / SP_CAP;
  for (int pass = 0; pass < (npass > 0 ? npass : 1); ++pass) {
    const int nk = (npass > 0) ? min(SP_CAP, r.xcnt - pass * SP_CAP) : 0;
    const float2* xp = xsrc + pass * SP_CAP;
    for (int b = tid; b <= SP_NBF; b += S3_T) S.start[b] = 0;
    __syncthreads();
    // ---- fine-bucket counting sort of this pass's x into shared memory
    int fr[S3_PER];   // (fine bucket << 13) | rank inside the bucket, -1: none
    float2 xw[S3_PER];   // the pass's (z, w), read once and kept in registers until the scatter
    {
#pragma unroll
      for (int k = 0; k < S3_PER; ++k) {   // all loads in flight before the first use
        const int i = tid + k * S3_T;
        xw[k] = (i < nk) ? ldg_cg2(xp + i) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < S3_PER; ++k) {
        fr[k] = -1;
        if (tid + k * S3_T < nk) {
          const int b = fine_of<SP_NBF>(ucoord(xw[k].x, uoff, hscale), r.blo, r.fmul);
          fr[k] = (b << 13) | atomicAdd(&S.start[b], 1);   // rank < SP_CAP <= 8192
        }
      }
    }
    __syncthreads();
    {
      constexpr int PB = SP_NBF / S3_T;   // buckets per thread (2 or 4)
      int c[PB], loc = 0;
#pragma unroll
      for (int j = 0; j < PB; ++j) { c[j] = S.start[tid * PB + j]; loc += c[j]; }
      int total;
      int run = block_excl_scan<S3_T>(loc, S.wbuf, &total);
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        S.start[tid * PB + j] = run;
        S.se[tid * PB + j] = static_cast<unsigned>(run) | (static_cast<unsigned>(run + c[j]) << 16);
        run += c[j];
      }
      if (tid == 0) S.start[SP_NBF] = total;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < S3_PER; ++k)
      if (fr[k] >= 0) {
        SKS_CHECK(S.start[fr[k] >> 13] + (fr[k] & 8191) < nk);
        S.xs[S.start[fr[k] >> 13] + (fr[k] & 8191)] = xw[k];
      }
    __syncthreads();
    if (det) {   // deterministic mode: each bucket's (z, w) in value order (the counting sort's order depends on the
                 // shared atomics' timing; the bucket sums below are then taken in a fixed order); a bucket holds a
                 // handful of points, one thread sorts it by insertion
      for (int b = tid; b < SP_NBF; b += S3_T) {
        const int2 br = se_unpack(S.se[b]);
        for (int i = br.x + 1; i < br.y; ++i) {
          const float2 v = S.xs[i];
          int j = i - 1;
          while (j >= br.x && (S.xs[j].x > v.x || (S.xs[j].x == v.x && S.xs[j].y > v.y))) {
            S.xs[j + 1] = S.xs[j];
            --j;
          }
          S.xs[j + 1] = v;
        }
      }
      __syncthreads();
    }
    // ---- fp64 bucket sums (thread t: buckets t, t + S3_T, ...: neighbouring lanes read neighbouring buckets)
    //      into rec[], then one blocked exclusive scan (thread t: buckets 4t .. 4t+3)
    double vc = 0.0;   // sum w z^2 of this thread's buckets (per-warp partials, summed by thread 0 below)
#pragma unroll
    for (int c0 = 0; c0 < SP_NBF; c0 += S3_T) {
      const int b = c0 + tid;
      double2 v = make_double2(0.0, 0.0);
      const int2 br = se_unpack(S.se[b]);
      for (int i = br.x, e = br.y; i < e; ++i) {
        const float2 q = S.xs[i];
        const double wz = static_cast<double>(q.y) * q.x;
        v.x += q.y;
        v.y += wz;
        vc += wz * q.x;
      }
      S.rec[b] = v;
    }
    vc = warp_sum_sp(vc);
    if ((tid & 31) == 0) wvc[tid >> 5] = vc;
    __syncthreads();
    {
      constexpr int PB = SP_NBF / S3_T;
      double2 v[PB], loc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < PB; ++j) { v[j] = S.rec[tid * PB + j]; loc = loc + v[j]; }
      double2 tch;
      double2 run = block_excl_scan_d2<S3_T>(loc, S.dbuf, &tch);
#pragma unroll
      for (int j = 0; j < PB; ++j) { S.rec[tid * PB + j] = run; run = run + v[j]; }
      if (tid == 0) {
        S.rec[SP_NBF] = tch;
        own_tot[0] += tch.x;
        own_tot[1] += tch.y;
        double c2 = 0.0;
#pragma unroll
        for (int q = 0; q < S3_T / 32; ++q) c2 += wvc[q];
        own_tot[2] += c2;
      }
    }
    __syncthreads();
    // ---- targets of this owner, all lookups in shared memory:
    //   sum_n w|x - z| = z(2A_b - A) - 2B_b + B + 2 sum_{x in b, x < z} w (z - x) + [other owners]
    const double2 Tp = S.rec[SP_NBF];
    constexpr int YB = MINB >= 3 ? 4 : 8;   // targets per thread per batch (register budget); next batch loads first
    float zn[YB];
#pragma unroll
    for (int k = 0; k < YB; ++k) {
      const int i = tid + k * S3_T;
      zn[k] = (i < r.ycnt) ? ldg_cg(ysrc + i) : 0.f;
    }
    for (int i0 = 0; i0 < r.ycnt; i0 += YB * S3_T) {
      float zy[YB];
#pragma unroll
      for (int k = 0; k < YB; ++k) zy[k] = zn[k];
#pragma unroll
      for (int k = 0; k < YB; ++k) {
        const int i = i0 + YB * S3_T + tid + k * S3_T;
        zn[k] = (i < r.ycnt) ? ldg_cg(ysrc + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < YB; ++k) {
        const int i = i0 + tid + k * S3_T;
        if (i >= r.ycnt) continue;
        const float zf = zy[k];
        const int b = fine_of<SP_NBF>(ucoord(zf, uoff, hscale), r.blo, r.fmul);
        const double2 rb = S.rec[b];
        const int2 jr = se_unpack(S.se[b]);
        const int j0 = jr.x, j1 = jr.y;
        float s0 = 0.f, s1 = 0.f;
        int j = j0;
        for (; j + 2 <= j1; j += 2) {
          const float2 q0 = S.xs[j], q1 = S.xs[j + 1];
          s0 = fmaf(q0.y, fmaxf(zf - q0.x, 0.f), s0);
          s1 = fmaf(q1.y, fmaxf(zf - q1.x, 0.f), s1);
        }
        if (j < j1) {
          const float2 q = S.xs[j];
          s0 = fmaf(q.y, fmaxf(zf - q.x, 0.f), s0);
        }
        const double zd = zf;
        // this owner's part only; the other owners' part is added in k_sp_gather (its other-owner table)
        const double v = zd * (2.0 * rb.x - Tp.x) - 2.0 * rb.y + Tp.y + 2.0 * static_cast<double>(s0 + s1);
        const float t = static_cast<float>(-coef * v);
        if (pass == 0) rdst[i] = t;
        else rdst[i] += t;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {   // publish this owner's x totals (the last pass ended with a barrier)
    double* ot = otot + (static_cast<int64_t>(p) * G + o) * 4;
    ot[0] = own_tot[0];
    ot[1] = own_tot[1];
    ot[2] = own_tot[2];
  }
}

// ---------------------------------------------------------------------------------------------- S4
// Many owners (G > kSmemDabMax): the other-owner table once per slice in global memory (k_sp_outer) instead of
// being rebuilt in every gather CTA's shared memory.
constexpr int SO_T = 256;

__global__ void __launch_bounds__(SO_T) k_sp_outer(const double* __restrict__ otot, int G, double2* __restrict__ dab,
                                                   SliceTot* __restrict__ tot) {
  __shared__ double wsc[3][SO_T / 32 + 1];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* ot = otot + static_cast<int64_t>(p) * G * 4;
  double carryA = 0.0, carryB = 0.0, carryC = 0.0;
  // totals first (two sweeps keep the code simple; G is small)
  for (int o0 = 0; o0 < G; o0 += SO_T) {
    const int o = o0 + tid;
    double a = 0.0, b = 0.0, c = 0.0;
    if (o < G) { a = ot[4 * o]; b = ot[4 * o + 1]; c = ot[4 * o + 2]; }
    a = warp_sum_sp(a); b = warp_sum_sp(b); c = warp_sum_sp(c);
    if (lane == 0) { wsc[0][wid] = a; wsc[1][wid] = b; wsc[2][wid] = c; }
    __syncthreads();
    if (tid == 0)
      for (int q = 0; q < SO_T / 32; ++q) { carryA += wsc[0][q]; carryB += wsc[1][q]; carryC += wsc[2][q]; }
    __syncthreads();
  }
  __shared__ double TA, TB;
  if (tid == 0) { TA = carryA; TB = carryB; tot[p] = SliceTot{carryA, carryB, carryC, 0.0}; }
  __syncthreads();
  const double A = TA, B = TB;
  double runA = 0.0, runB = 0.0;   // exclusive prefix over owner chunks
  for (int o0 = 0; o0 < G; o0 += SO_T) {
    const int o = o0 + tid;
    double a = 0.0, b = 0.0;
    if (o < G) { a = ot[4 * o]; b = ot[4 * o + 1]; }
    double ia = warp_incl_scan_sp(a), ib = warp_incl_scan_sp(b);
    if (lane == 31) { wsc[0][wid] = ia; wsc[1][wid] = ib; }
    __syncthreads();
    double wa = 0.0, wb = 0.0, ta = 0.0, tb = 0.0;
    for (int q = 0; q < SO_T / 32; ++q) {
      if (q < wid) { wa += wsc[0][q]; wb += wsc[1][q]; }
      ta += wsc[0][q];
      tb += wsc[1][q];
    }
    const double alo = runA + wa + ia - a, blo = runB + wb + ib - b;   // owners < o
    if (o < G) dab[static_cast<int64_t>(p) * G + o] = make_double2(alo - (A - alo - a), (B - blo - b) - blo);
    runA += ta;
    runB += tb;
    __syncthreads();
  }
}

static_assert(S4_SG == S4_T / 32, "one warp per slice of the gather's slice group builds its other-owner table");

template <bool GDAB>
__global__ void __launch_bounds__(S4_T) k_sp_gather(ZView zv, int np, int G, double coef, const int* __restrict__ ypos,
                                                    const uint16_t* __restrict__ yown, const float* __restrict__ R,
                                                    const double* __restrict__ otot, SliceTot* __restrict__ tot,
                                                    const double2* __restrict__ gdab, TargetAcc tacc,
                                                    float* __restrict__ per_slice_out) {
  extern __shared__ double2 sdab[];   // [S4_SG][G] other-owner coefficients of the group's slices (gdab == null)
  const int64_t M = zv.M;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * S4_CH + threadIdx.x;
  const int p0 = blockIdx.y * S4_SG, p1 = min(np, p0 + S4_SG);
  {
    // warp w: slice p0 + w.  For a target of owner o, the x of owners < o lie below it and those of owners > o
    // above it: sum w |x - z| over them = z (Alo - Ahi) + (Bhi - Blo), from the owners' fp64 totals (fused here:
    // every CTA of the slice group rebuilds the small table; the first target block also writes the slice totals)
    const int wid = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;   // (uniform)
    const int p = p0 + wid;
    if (p < p1 && !GDAB) {
      const double* ot = otot + static_cast<int64_t>(p) * G * 4;
      double A = 0.0, B = 0.0, C = 0.0;
      for (int o = lane; o < G; o += 32) { A += ot[4 * o]; B += ot[4 * o + 1]; C += ot[4 * o + 2]; }
      A = warp_sum_sp(A); B = warp_sum_sp(B); C = warp_sum_sp(C);
      if (blockIdx.x == 0 && lane == 0) tot[p] = SliceTot{A, B, C, 0.0};
      double runA = 0.0, runB = 0.0;
      for (int o0 = 0; o0 < G; o0 += 32) {
        const int o = o0 + lane;
        const double a = o < G ? ot[4 * o] : 0.0, b = o < G ? ot[4 * o + 1] : 0.0;
        const double ia = warp_incl_scan_sp(a), ib = warp_incl_scan_sp(b);
        const double alo = runA + ia - a, blo = runB + ib - b;   // owners < o
        if (o < G) sdab[wid * G + o] = make_double2(alo - (A - alo - a), (B - blo - b) - blo);
        runA += __shfl_sync(0xffffffffu, ia, 31);
        runB += __shfl_sync(0xffffffffu, ib, 31);
      }
    }
    __syncthreads();
  }
  double acc[S4_PER];
#pragma unroll
  for (int k = 0; k < S4_PER; ++k) acc[k] = 0.0;
  for (int p = p0; p < p1; ++p) {
    int q[S4_PER], ow[S4_PER];
    float z[S4_PER];
#pragma unroll
    for (int k = 0; k < S4_PER; ++k) {
      const int64_t m = m0 + k * S4_T;
      const bool ok = m < M;
      q[k] = ok ? __ldcs(ypos + static_cast<int64_t>(p) * M + m) : 0;
      ow[k] = ok ? yown[static_cast<int64_t>(p) * M + m] : 0;
      z[k] = ok ? __ldg(zv.zy + p * zv.ldy + m) : 0.f;
    }
    float t[S4_PER];
    double2 d[S4_PER];
#pragma unroll
    for (int k = 0; k < S4_PER; ++k) {
      const int64_t m = m0 + k * S4_T;
      t[k] = (m < M) ? __ldcs(R + static_cast<int64_t>(p) * M + q[k]) : 0.f;
      d[k] = (m < M) ? (GDAB ? __ldg(gdab + static_cast<int64_t>(p) * G + ow[k]) : sdab[(p - p0) * G + ow[k]])
                     : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < S4_PER; ++k) {
      const int64_t m = m0 + k * S4_T;
      if (m >= M) continue;
      const double tt = static_cast<double>(t[k]) - coef * (static_cast<double>(z[k]) * d[k].x + d[k].y);
      acc[k] += tt;
      if (per_slice_out) per_slice_out[static_cast<int64_t>(p) * M + m] = static_cast<float>(tt);
    }
  }
#pragma unroll
  for (int k = 0; k < S4_PER; ++k) {
    const int64_t m = m0 + k * S4_T;
    if (m < M) acc_target(tacc, blockIdx.y, m, acc[k]);
  }
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// histogram chunks of a slice part: S0_CH elements each, at most 8 chunks, then longer chunks (measured
// N = 1e6 / 1e7, P = 1000: at most 8 -> 34.4 / 528 ms, 16 -> 36.0 / 528, 32 -> 38.6 / 526)
constexpr int kHistMaxChunks = 8;
inline int hist_chunks(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kHistMaxChunks, cdiv(n, S0_CH))));
}
inline int hist_chunk_len(int64_t n) { return static_cast<int>(std::max<int64_t>(1, cdiv(n, hist_chunks(n)))); }

}  // namespace

SpDims sortpart_dims(int64_t N, int64_t M) {
  SpDims d;
  // histogram bins: ~64 x per bin on average (owners of ~3000 x balance to a bin), at least 2048, at most 16384
  // (u16 owner map in shared memory)
  int nh = 2048;
  while (nh < 16384 && static_cast<int64_t>(nh) * 64 < N) nh *= 2;   // (32 / 64 / 128 per bin measured: 64)
  d.NH = nh;
  // owners: 85% of the owner capacity each (room for the bin granularity of the balance)
  int64_t g = cdiv(N, SP_CAP * 85 / 100);   // (60 / 75 / 85 / 95% measured: 85-95 best, 85 leaves room)
  if (g < 1) g = 1;
  if (g > 4096) g = 4096;   // (u16 owner ids; beyond, owners take several passes)
  d.G = static_cast<int>(g);
  (void)M;
  return d;
}

// The slices are processed in groups, the groups round-robin on kSortStreams streams forked from the caller's
// stream, each stream with its own scratch region: the four kernels of one group are latency-bound at their
// phase boundaries, and a second group's kernels fill the idle SMs (1 -> 2 streams: cfg2 1.11 -> 1.03 ms; 3 / 4
// no better).  Group size ceil(P_batch / streams) (measured 4 / 12 / 48 / 256 slices on one stream: 7.2 / 3.2 /
// 1.49 / 0.95 ms on cfg2: the per-group tails dominate small groups).
constexpr int kSortStreams = 2;
int sortpart_streams() { return kSortStreams; }

int sortpart_group(int64_t N, int64_t M, int np) {
  (void)N;
  (void)M;
  const int64_t g = (np + kSortStreams - 1) / kSortStreams;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, np)));
}

static size_t region_bytes(int64_t N, int64_t M, int np) {
  const SpDims d = sortpart_dims(N, M);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  size_t s = 0;
  s += al(sizeof(int) * (hist_chunks(N) + hist_chunks(M)) * d.NH * static_cast<size_t>(np));   // H (per chunk)
  s += al(sizeof(int) * 2 * d.G * static_cast<size_t>(np));           // cursors
  s += al(sizeof(int) * static_cast<size_t>(np));                     // done tickets
  s += al(sizeof(double) * 4 * d.G * static_cast<size_t>(np));        // owner totals
  s += al(sizeof(double2) * d.G * static_cast<size_t>(np));           // other-owner coefficients (large G)
  s += al(sizeof(int) * (hist_chunks(N) + hist_chunks(M)) * d.G * static_cast<size_t>(np));   // (chunk, owner) bases
  s += al(sizeof(uint16_t) * M * static_cast<size_t>(np));            // y owners
  s += al(sizeof(uint16_t) * d.NH * static_cast<size_t>(np));         // owner map
  s += al(sizeof(SpOwner) * d.G * static_cast<size_t>(np));           // owners
  s += al(sizeof(float2) * N * static_cast<size_t>(np));              // x mailbox
  s += al(sizeof(float) * M * static_cast<size_t>(np));               // y mailbox
  s += al(sizeof(float) * M * static_cast<size_t>(np));               // results
  s += al(sizeof(int) * M * static_cast<size_t>(np));                 // y positions
  return s;
}

static int active_streams(int64_t N, int64_t M, int np) {
  const int gs = sortpart_group(N, M, np);
  return std::min(sortpart_streams(), (np + gs - 1) / gs);
}

int sortpart_acc_groups(int64_t N, int64_t M, int np) {
  const int gs = sortpart_group(N, M, np);
  return static_cast<int>(cdiv(np, gs) * cdiv(gs, S4_SG));
}

int sortpart_launches_per_group(int64_t N, int64_t M) { return sortpart_dims(N, M).G > kSmemDabMax ? 5 : 4; }

size_t sortpart_bytes(int64_t N, int64_t M, int np) {
  return region_bytes(N, M, sortpart_group(N, M, np)) * active_streams(N, M, np);
}

namespace {
// helper streams and fork / join events: one set per (thread, device), so that concurrent calls on different
// threads never share an event, and a call on another device never launches onto this device's streams
struct StreamPool {
  cudaStream_t s[kSortStreams] = {};
  cudaEvent_t fork = nullptr, join[kSortStreams] = {};
  bool ok = false;
};
StreamPool& stream_pool(int dev) {
  thread_local std::map<int, StreamPool> pools;
  StreamPool& pool = pools[dev];
  if (!pool.ok) {
    bool good = cudaEventCreateWithFlags(&pool.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 1; i < kSortStreams && good; ++i)
      good = cudaStreamCreateWithFlags(&pool.s[i], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&pool.join[i], cudaEventDisableTiming) == cudaSuccess;
    pool.ok = good;
  }
  return pool;
}
}  // namespace

namespace {
// scratch of one slice group (one region per stream; regions are reused by the groups of that stream)
struct SpRegion {
  int* cursor;      // [gs][2][G] mailbox cursors       } zeroed per group
  int* done;        // [gs] histogram tickets           }
  size_t zero_bytes;
  int* H;           // [gs][chunks][NH] chunk histograms
  double* otot;     // [gs][G][4] owner totals (w, w z, w z^2)
  double2* dab;     // [gs][G] other-owner coefficients (G > kSmemDabMax only)
  int* base;        // [gs][chunks][G] first mailbox slot of every (chunk, owner) (G > kSmemDabMax only)
  uint16_t* yown;   // [gs][M] owner of each target
  uint16_t* om;     // [gs][NH] owner of each bin
  SpOwner* own;     // [gs][G]
  float2* Xmb;      // [gs][N] x mailbox (z, w)
  float* Ymb;       // [gs][M] y mailbox (z)
  float* R;         // [gs][M] own-owner part of t, mailbox order
  int* ypos;        // [gs][M] mailbox slot of each target
};

SpRegion carve_region(char* base, int64_t N, int64_t M, int NH, int G, int gs) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t g = static_cast<size_t>(gs);
  SpRegion r;
  char* w = base;
  r.cursor = reinterpret_cast<int*>(w);       w += al(sizeof(int) * 2 * G * g);
  r.done = reinterpret_cast<int*>(w);         w += al(sizeof(int) * g);
  r.zero_bytes = static_cast<size_t>(w - base);
  r.H = reinterpret_cast<int*>(w);            w += al(sizeof(int) * (hist_chunks(N) + hist_chunks(M)) * NH * g);
  r.otot = reinterpret_cast<double*>(w);      w += al(sizeof(double) * 4 * G * g);
  r.dab = reinterpret_cast<double2*>(w);      w += al(sizeof(double2) * G * g);
  r.base = reinterpret_cast<int*>(w);         w += al(sizeof(int) * (hist_chunks(N) + hist_chunks(M)) * G * g);
  r.yown = reinterpret_cast<uint16_t*>(w);    w += al(sizeof(uint16_t) * M * g);
  r.om = reinterpret_cast<uint16_t*>(w);      w += al(sizeof(uint16_t) * NH * g);
  r.own = reinterpret_cast<SpOwner*>(w);      w += al(sizeof(SpOwner) * G * g);
  r.Xmb = reinterpret_cast<float2*>(w);       w += al(sizeof(float2) * N * g);
  r.Ymb = reinterpret_cast<float*>(w);        w += al(sizeof(float) * M * g);
  r.R = reinterpret_cast<float*>(w);          w += al(sizeof(float) * M * g);
  r.ypos = reinterpret_cast<int*>(w);
  return r;
}

// dynamic shared-memory limits: a function attribute is per device, so it is set once per device
void set_attributes(int dev) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return;
  cudaFuncSetAttribute(k_sp_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);   // (+ static shared)
  cudaFuncSetAttribute(k_sp_part, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_sp_part_big<S0_T, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_sp_part_big<S0_T, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_sp_part_big<1024, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_sp_gather<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_sp_owner<SP_CAP, SP_NBF, SP_MINB, SP_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(sizeof(OwnerShared<SP_CAP, SP_NBF, SP_NT>)));
  done.insert(dev);
}

// elements per thread of a k_sp_part_big sub-chunk: measured N = 1e7, P = 100 sort stage (ms, {G cap, per thread}):
// {1024, 8} 51.3, {4096, 8} 58.2, {4096, 16} 49.1, {2048, 16} 49.4; N = 3e6 (G = 862): 8 -> 10.89, 16 -> 11.02.  More
// owners shorten the owner passes and the gather (26.9 -> 17.4 ms) but cut the mailbox runs per sub-chunk, so the
// sub-chunk grows with G.
int part_sbper(int G) { return G > 1024 ? 16 : 8; }

// threads of a k_sp_part_big CTA (1024: 8 elements per thread, the same 8192-element sub-chunk as 512 x 16 at
// twice the warps per SM -- the kernel is latency bound at one CTA per SM, ncu: 25% of the warp slots active).
// Measured N = 1e7, P = 100 / 1000: 512 x 16 53.4 / 529 ms, 1024 x 8 49.4 / 489; N = 1e6 (288 owners): no difference.
int part_big_threads(int G) { return G > 1024 ? 1024 : S0_T; }

// the five kernels of one slice group (slices [g0, g0 + np) of the call) on stream st
cudaError_t launch_group(const SortPartArgs& a, const SpRegion& r, int gi, int g0, int np, int NH, int G,
                         cudaStream_t st) {
  const int64_t N = a.zv.N, M = a.zv.M;
  constexpr int wpc = 8;   // partition: 256-element rounds per warp (measured 4: 0.850, 8: 0.835, 16: 0.834 ms cfg2)
  const int ncx0 = hist_chunks(N), ncy0 = hist_chunks(M);
  const int64_t per_cta2 = int64_t(S2W_WARPS) * S2W_WCH * wpc;
  const int ncx2 = static_cast<int>(cdiv(N, per_cta2)), ncy2 = static_cast<int>(cdiv(M, per_cta2));
  // many owners: plan bases + atomic-free partition (k_sp_part_big); with few (cfg2: 29) the warp rounds win
  // (measured with the big path forced at G = 29: cfg2 0.817 -> 0.846 ms)
  const bool big = G > kSmemDabMax;
  const int nch = ncx0 + ncy0;
  // plan bases: every chunk at once while cnt[nch][G] fits (measured N = 1e6, G = 288: one chunk at a time is
  // 2% slower), else one chunk at a time
  const size_t plan_ints = 2 * (NH + 1) + G + 1;
  const int base_par = big && plan_ints + static_cast<size_t>(nch) * G <= 200 * 1024 / sizeof(int);
  const size_t sm0 = sizeof(int) * std::max<size_t>(
      NH, plan_ints + (big ? (base_par ? static_cast<size_t>(nch) * G : 3 * static_cast<size_t>(G)) : 0));
  const size_t sm2 = sizeof(int) * (((1 + S2W_WARPS) * G + 3) / 4 * 4) + sizeof(uint16_t) * NH;
  const int sbper = part_sbper(G);
  const int sbelems = part_big_threads(G) == 1024 ? 1024 * 8 : S0_T * sbper;
  const size_t sm2b = sizeof(int) * 2 * ((G + 3) / 4 * 4) + (sizeof(float2) + sizeof(uint16_t)) * sbelems +
                      sizeof(uint16_t) * NH;
  ZView zv = a.zv;
  zv.zx += g0 * zv.ldx;
  zv.zy += g0 * zv.ldy;
  const unsigned* mm = a.mm + 4 * g0;
  float* pso = a.per_slice_out ? a.per_slice_out + static_cast<int64_t>(g0) * M : nullptr;
  cudaError_t e = cudaMemsetAsync(r.cursor, 0, r.zero_bytes, st);
  if (e != cudaSuccess) return e;
  ProfMark pm = prof_begin(PS_SP_HIST, st);
  k_sp_hist<<<dim3(ncx0 + ncy0, np), S0_T, sm0, st>>>(zv, mm, NH, G, ncx0, ncx0 + ncy0, hist_chunk_len(N),
                                                       hist_chunk_len(M), SP_NBF, r.H, r.done, r.om,
                                                       r.own, big ? r.base : nullptr, base_par);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  prof_end(pm);
  pm = prof_begin(PS_SP_PART, st);
  if (big)
  {
    const int pbt = part_big_threads(G);
    auto kern = pbt == 1024 ? k_sp_part_big<1024, 8> : (sbper == 16 ? k_sp_part_big<S0_T, 16> : k_sp_part_big<S0_T, 8>);
    kern<<<dim3(nch, np), pbt, sm2b, st>>>(zv, a.w, mm, NH, G, ncx0, nch, hist_chunk_len(N), hist_chunk_len(M), r.om,
                                           r.base, r.Xmb, r.Ymb, r.ypos, r.yown);
  }
  else
    k_sp_part<<<dim3(ncx2 + ncy2, np), S2W_T, sm2, st>>>(zv, a.w, mm, NH, G, ncx2, wpc, r.om, r.own, r.cursor, r.Xmb,
                                                          r.Ymb, r.ypos, r.yown);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  prof_end(pm);
  pm = prof_begin(PS_SP_OWNER, st);
  k_sp_owner<SP_CAP, SP_NBF, SP_MINB, SP_NT><<<dim3(G, np), SP_NT, sizeof(OwnerShared<SP_CAP, SP_NBF, SP_NT>), st>>>(
      r.own, r.otot, mm, NH, G, N, M, r.Xmb, r.Ymb, a.coef, r.R, a.det ? 1 : 0);
  prof_end(pm);
  pm = prof_begin(PS_SP_GATHER, st);
  const bool smem_dab = G <= kSmemDabMax;   // few owners: each gather CTA builds its slices' table in shared memory
  if (!smem_dab) k_sp_outer<<<np, SO_T, 0, st>>>(r.otot, G, r.dab, a.tot + g0);
  const dim3 ggrid(static_cast<unsigned>(cdiv(M, S4_CH)), static_cast<unsigned>(cdiv(np, S4_SG)));
  TargetAcc tacc = a.acc;   // this group's rows of the TargetAcc groups (deterministic mode)
  tacc.goff += gi * static_cast<int>(cdiv(sortpart_group(N, M, a.np), S4_SG));
  if (smem_dab)
    k_sp_gather<false><<<ggrid, S4_T, sizeof(double2) * S4_SG * G, st>>>(zv, np, G, a.coef, r.ypos, r.yown, r.R, r.otot,
                                                                        a.tot + g0, nullptr, tacc, pso);
  else
    k_sp_gather<true><<<ggrid, S4_T, 0, st>>>(zv, np, G, a.coef, r.ypos, r.yown, r.R, r.otot, a.tot + g0, r.dab,
                                              tacc, pso);
  prof_end(pm);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_sortpart(const SortPartArgs& a, void* ws, cudaStream_t st) {
  const int64_t N = a.zv.N, M = a.zv.M;
  const SpDims d = sortpart_dims(N, M);
  const int gs = sortpart_group(N, M, a.np);
  const int ns = active_streams(N, M, a.np);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  set_attributes(dev);
  StreamPool& pool = stream_pool(dev);
  if (ns > 1 && !pool.ok) return cudaErrorInitializationError;
  if (ns > 1) {   // fork: the helper streams start after everything already queued on the caller's stream
    if ((e = cudaEventRecord(pool.fork, st)) != cudaSuccess) return e;
    for (int i = 1; i < ns; ++i)
      if ((e = cudaStreamWaitEvent(pool.s[i], pool.fork, 0)) != cudaSuccess) return e;
  }
  const size_t rb = region_bytes(N, M, gs);
  for (int g0 = 0, gi = 0; g0 < a.np; g0 += gs, ++gi) {
    const int si = gi % ns;
    const SpRegion r = carve_region(static_cast<char*>(ws) + rb * si, N, M, d.NH, d.G, gs);
    if ((e = launch_group(a, r, gi, g0, std::min(gs, a.np - g0), d.NH, d.G, si ? pool.s[si] : st)) != cudaSuccess)
      return e;
  }
  for (int i = 1; i < ns; ++i) {   // join
    if ((e = cudaEventRecord(pool.join[i], pool.s[i])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, pool.join[i], 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sks
