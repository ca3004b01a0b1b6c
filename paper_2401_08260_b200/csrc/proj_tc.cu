// proj_tc.cu -- row a1 on the 5th-generation tensor cores: the projection Z[p][i] = <xi_p, z_i> (P:129,
// Alg. 1) as one bf16 GEMM with fp32 accumulation that is fp32-accurate (reading R2):
//   * directions g_p are bf16-exact by construction (R1), xi_p = g_p / ||g_p|| is applied in the epilogue;
//   * each fp32 coordinate is split exactly-enough into three bf16 pieces x = hi + mid + lo (+ O(2^-24 |x|)),
//     stored K-concatenated: Xs[i] = [hi(0..dp) | mid(0..dp) | lo(0..dp)], G3[p] = [g_p | g_p | g_p];
//   * every bf16 x bf16 product is exact in fp32, so D = Xs . G3^T is <g_p, x_i> with fp32 accumulation.
// Kernel: TMA (cp.async.bulk.tensor, 128B swizzle) -> smem ring -> tcgen05.mma.cta_group::1.kind::f16
// (M=128 points x N=BN slices x K=16) accumulating in TMEM -> tcgen05.ld epilogue (scale by 1/||g_p||,
// coalesced stores along points, per-slice x / all ranges, non-finite flag).  Warp roles: w0 TMA producer,
// w1 MMA issuer, w2 TMEM allocator, w4..w7 epilogue (TMEM lane quadrants 0..3).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "tc_util.h"

namespace sks {

namespace {

using namespace tc;

constexpr int TC_M = 128;   // points per tile (UMMA M)
constexpr int TC_BK = 64;   // bf16 elements per k-block = 128 bytes (one swizzle row)
constexpr int kProjMaxCtas = 148;   // persistent grid: one CTA per SM

__device__ __forceinline__ unsigned f2key_tc(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// FP16x2 point scale s = 2^(14 - e), max|x| = m 2^e (m in [0.5, 1)): s max|x| < 2^14 (1 if max|x| = 0)
__device__ __forceinline__ float f16_scale(unsigned maxbits) {
  const float m = __uint_as_float(maxbits);
  if (!(m > 0.f) || !(m < 3.0e38f)) return 1.0f;
  int e;
  frexpf(m, &e);
  return ldexpf(1.0f, 14 - e);
}

// max |x| over a sample of the points (rows k L / S, k < S; d % 4 == 0, 16-byte aligned rows) into *out (float bits; positive floats order as
// unsigned ints), for the FP16x2 scale; out zeroed by the caller
__global__ void k_absmax_sample(const float* __restrict__ x, int64_t N, const float* __restrict__ y, int64_t M, int d,
                                int S, unsigned* __restrict__ out) {
  const int64_t L = N + M;
  float m = 0.f;
  for (int k = blockIdx.x; k < S; k += gridDim.x) {   // one row per CTA and step, 16-byte loads (d % 4 == 0)
    const int64_t i = static_cast<int64_t>(k) * L / S;
    const float4* row = reinterpret_cast<const float4*>((i < N) ? x + i * d : y + (i - N) * d);
    for (int j = threadIdx.x; j < d / 4; j += blockDim.x) {
      const float4 v = __ldg(row + j);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// Stage of the k-loop.  BF16x3 (TF32 = false): three bf16 pieces of 128 points x 64 dims (TMA from the split
// buffer) + the direction tile.  TF32x2 (TF32 = true): hi / lo tf32 pieces of 128 points x 32 dims written by
// the converter warps straight from the fp32 points + the fp32 direction tile (TMA).  Rows are 128 bytes,
// 128-byte swizzled, in both cases.
// MODE 0: BF16x3 from the pre-split buffer (TMA); 1: TF32x2 (raw fp32 points = hi operand, converters form
// lo); 3: FP16x2 (raw fp32 points by TMA into the hi / lo slots, converters write fp16 hi / lo of the scaled
// points in place; directions as fp16 x 2^8)
template <int BN, int STAGES, int MODE = 0>
struct TcSmem {
  static constexpr bool TF32 = MODE == 1;
  static constexpr int NPIECE = MODE == 0 ? 3 : 2;
  static constexpr int A_BYTES = TC_M * 128;                // one piece: 128 points x 128 bytes
  static constexpr int B_BYTES = BN * 128;                  // BN directions x 128 bytes
  static constexpr int STAGE = NPIECE * A_BYTES + B_BYTES;  // the pieces share one direction tile
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int RANGE_OFF = (BAR_OFF + 8 * (3 * STAGES + 4) + 16 + 63) / 64 * 64;   // float4-aligned
  static constexpr int FIXED = RANGE_OFF + 1024;            // + per-CTA range partials [np_pad][4], 1/||g|| + slack
};

// min / max of 16 columns (fmn[j] / fmx[j] = this lane's value of column j) over the 32 lanes of a warp by warp
// reductions (redux.sync f32, sm_100a): lane j (< 16) gets column j's bounds (finite inputs; NaN / Inf are trapped
// separately)
__device__ __forceinline__ void colrange16r(const float* fmn, const float* fmx, int lane, float* omn, float* omx) {
  float mn = CUDART_INF_F, mx = -CUDART_INF_F;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float a, b;
    asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(a) : "f"(fmn[j]));
    asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(b) : "f"(fmx[j]));
    mn = lane == j ? a : mn;
    mx = lane == j ? b : mx;
  }
  *omn = mn;
  *omx = mx;
}

// Persistent: grid = min(#tiles, #SMs) CTAs, tiles t = blockIdx.x + i*gridDim.x (slice tiles fastest, so the
// CTAs that share a point tile run together and its TMA loads hit L2).  Two TMEM accumulators: the epilogue
// of tile i overlaps the MMAs of tile i+1.  Per-slice ranges: per-CTA partials in smem -> global atomics.
constexpr int TC_THREADS = 384;   // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4..w11 epilogue (2 warpgroups)
constexpr int TC_THREADS_TF32 = 512;   // + converter warps (TF32x2: w12..w15; FP16x2: w8..w15, 4 epilogue warps)

// round to the nearest tf32 (10 explicit mantissa bits), kept in an fp32 container: exact tensor-core operand
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

template <int BN, int STAGES, int MODE = 0>
__global__ void __launch_bounds__(MODE != 0 ? TC_THREADS_TF32 : TC_THREADS, 1)
    k_proj_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int nk, int64_t L,
              int64_t Nx, int np, const float* __restrict__ inv_norm, float* __restrict__ Z, int64_t ldz,
              unsigned* __restrict__ mm, int* __restrict__ flag, const float* __restrict__ px,
              const float* __restrict__ py, int d, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmY, int xtma, const unsigned* __restrict__ f16max,
              const unsigned* __restrict__ pred) {
  if (pred && *pred == 0) return;   // predicated launch (the FP16x2 -> TF32x2 rerun): nothing to redo
  using SM = TcSmem<BN, STAGES, MODE>;
  constexpr bool TF32 = MODE == 1, CONV = MODE != 0, F16 = MODE == 3;
  // warp roles: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle; epilogue warps 4 .. 4 + NEPI - 1; converters CW0 .. 15.
  // FP16x2 (tensor-bound, d >= 256) trades epilogue warps for converters: 4 epilogue warps (all columns of a
  // lane quadrant each) and 8 converter warps (16 rows each)
  constexpr int NEPI = F16 ? 4 : 8, CW0 = F16 ? 8 : 12, NCONV = 16 - CW0, RPW = TC_M / NCONV;
  extern __shared__ unsigned char smraw[];
  // aligned by pointer arithmetic on the __shared__ array: the compiler keeps the shared state space (LDS / STS,
  // not generic LD / ST)
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + SM::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;     // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint64_t* xfull = tempty + 2;         // [STAGES] TF32x2 with TMA points: the raw fp32 tile (hi piece) landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + STAGES);
  unsigned* rng = reinterpret_cast<unsigned*>(sm + SM::RANGE_OFF);   // [np_pad][4] keys
  // (the warp index through a shuffle: visibly warp-uniform, so the role branches below are uniform and the
  // epilogue's warp collectives (redux, shuffles) compile without divergence handling)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int ntn = (np + BN - 1) / BN;
  float* sinv = reinterpret_cast<float*>(rng + 4 * ntn * BN);          // [np_pad] 1/||g_p||
  // FP16x2: D accumulates (2^8 g) . (s x); the epilogue scale takes 1 / (2^8 s) with the 1 / ||g||
  const float zs = F16 ? 1.0f / (256.0f * f16_scale(__ldg(f16max))) : 1.0f;
  for (int c = threadIdx.x; c < ntn * BN; c += blockDim.x) sinv[c] = (c < np) ? inv_norm[c] * zs : 0.f;
  const int64_t ntm = (L + TC_M - 1) / TC_M;
  const int64_t ntiles = ntm * ntn;
  for (int c = threadIdx.x; c < ntn * BN; c += blockDim.x) {
    rng[4 * c + 0] = 0xffffffffu; rng[4 * c + 1] = 0u; rng[4 * c + 2] = 0xffffffffu; rng[4 * c + 3] = 0u;
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], CONV ? NCONV + 1 : 1);
      mbar_init(&empty[s], 1);
      mbar_init(&xfull[s], 1);
    }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (CONV && xtma) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmY)) : "memory");
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m0 = static_cast<int>((t / ntn) * TC_M), n0 = static_cast<int>(t % ntn) * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* sa = sm + stage * SM::STAGE;
        if (F16) {   // raw fp32 points (two boxes of 32 dims) into the hi / lo slots + the fp16 direction tile
          const bool hasx = m0 < Nx;
          mbar_expect_tx(&xfull[stage], 2 * SM::A_BYTES);
          // a tile straddling x / y: the x rows by TMA (the rest zero-filled), the y rows by the converters
          const CUtensorMap* mp = hasx ? &tmX : &tmY;
          const int row = hasx ? static_cast<int>(m0) : static_cast<int>(m0 - Nx);
          tma_load_2d(mp, &xfull[stage], sa, kb * 64, row);
          tma_load_2d(mp, &xfull[stage], sa + SM::A_BYTES, kb * 64 + 32, row);
          mbar_expect_tx(&full[stage], SM::B_BYTES);
          tma_load_2d(&tmB, &full[stage], sa + 2 * SM::A_BYTES, kb * TC_BK, n0);
        } else if (TF32) {   // TMA brings the direction tile (and, with xtma, the raw fp32 points = the hi piece)
          if (xtma) {
            // rows m0 .. m0 + 127 of the concatenated points: x rows from tmX, y rows from tmY (rows outside a
            // map are zero-filled); a tile straddling x / y lands its y rows in the lo slot, merged by the converters
            const bool hasx = m0 < Nx, hasy = m0 + TC_M > Nx && L > Nx;
            mbar_expect_tx(&xfull[stage], (hasx && hasy ? 2 : 1) * SM::A_BYTES);
            if (hasx) tma_load_2d(&tmX, &xfull[stage], sa, kb * 32, m0);
            if (hasy) tma_load_2d(&tmY, &xfull[stage], hasx ? sa + SM::A_BYTES : sa, kb * 32, static_cast<int>(m0 - Nx));
          }
          mbar_expect_tx(&full[stage], SM::B_BYTES);
          tma_load_2d(&tmB, &full[stage], sa + 2 * SM::A_BYTES, kb * 32, n0);
        } else {
          mbar_expect_tx(&full[stage], SM::STAGE);
#pragma unroll
          for (int q = 0; q < 3; ++q) tma_load_2d(&tmA, &full[stage], sa + q * SM::A_BYTES, (q * nk + kb) * TC_BK, m0);
          tma_load_2d(&tmB, &full[stage], sa + 3 * SM::A_BYTES, kb * TC_BK, n0);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread)
    constexpr uint32_t idesc = TF32 ? idesc_tf32(TC_M, BN) : F16 ? idesc_f16(TC_M, BN) : idesc_bf16(TC_M, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      const uint32_t tph = (it >> 1) & 1;
      mbar_wait(&tempty[b], tph ^ 1);   // epilogue drained this accumulator
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(b * BN);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned char* sa = sm + stage * SM::STAGE;
        const uint64_t db = umma_desc_sw128(sa + SM::NPIECE * SM::A_BYTES);
#pragma unroll
        for (int q = 0; q < SM::NPIECE; ++q) {
          const uint64_t da = umma_desc_sw128(sa + q * SM::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {   // 4 MMAs of K = 32 bytes (16 bf16 / 8 tf32) per 128-byte row
            const uint32_t acc = (kb > 0 || q > 0 || k > 0) ? 1u : 0u;
            const uint64_t adv = static_cast<uint64_t>((k * 32) >> 4);   // +32 B along K inside the swizzle row
            if (TF32)
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                  "l"(da + adv), "l"(db + adv), "r"(idesc), "r"(acc));
            else
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
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&tfull[b]))
                   : "memory");
    }
  } else if (F16 && warp >= CW0) {
    // ---- converters (FP16x2): the raw fp32 rows of a k-block (64 dims) sit in the hi / lo slots (128-byte
    //      swizzled fp32 boxes of 32 dims).  Lane c of a 4-row group reads dims 8c .. 8c + 7 of its row (two
    //      16-byte fp32 chunks), the warp syncs, then writes fp16 chunk c of hi = f16(s x) and lo = f16(s x - hi)
    //      for that row (|s x - hi - lo| <= 2^-22 |s x| + 2^-25: the 22-bit precision of TF32x2).  s = 2^e puts
    //      the largest sampled |x| near 2^14; a value beyond the fp16 range (|s x| >= 65520, outside the sample)
    //      becomes Inf and trips the epilogue's non-finite trap: the caller reruns the call with TF32x2, which
    //      reports genuine NaN / Inf inputs.  Rows are private to a warp (RPW = 16 rows per converter warp).
    const int cw = warp - CW0;
    const int c = lane & 7, rsub = lane >> 3;
    const float xs = f16_scale(__ldg(f16max));
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t m0 = (t / ntn) * TC_M;
      const int split = (m0 < Nx && m0 + TC_M > Nx) ? static_cast<int>(Nx - m0) : TC_M;   // y rows >= split
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&xfull[stage], phase);
        unsigned char* sa = sm + stage * SM::STAGE;
        // two halves of 4 row groups: all 4 groups' raw chunks are read before the warp syncs and overwrites them
#pragma unroll
        for (int hb = 0; hb < RPW / 4; hb += 4) {
          float v[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = RPW * cw + 4 * (hb + q) + rsub;
            const int box = c >> 2, j0 = 2 * (c & 3);   // fp32 box (0: hi slot, 1: lo slot), chunks j0, j0 + 1
            const unsigned char* rb = sa + box * SM::A_BYTES + r * 128;
            if (r < split) {
              // the two boxes are 16 KB apart (same banks): lanes of box 1 read their two chunks in the other
              // order, so that the 8 lanes of a quarter-warp hit 8 distinct 16-byte bank groups per load
              const int jf = j0 + box, js = j0 + 1 - box;
              const float4 f4 = *reinterpret_cast<const float4*>(rb + ((jf ^ (r & 7)) << 4));
              const float4 s4 = *reinterpret_cast<const float4*>(rb + ((js ^ (r & 7)) << 4));
              const float4 a4 = box ? s4 : f4, b4 = box ? f4 : s4;
              v[q][0] = a4.x; v[q][1] = a4.y; v[q][2] = a4.z; v[q][3] = a4.w;
              v[q][4] = b4.x; v[q][5] = b4.y; v[q][6] = b4.z; v[q][7] = b4.w;
            } else {   // straddling tile: y rows from global memory
              const int64_t i = m0 + r;
              const int col = kb * 64 + 8 * c;
#pragma unroll
              for (int u = 0; u < 8; ++u) v[q][u] = 0.f;
              if (i < L) {
                const float* row = py + (i - Nx) * static_cast<int64_t>(d);
                if (col < d) {
                  const float4 a4 = __ldg(reinterpret_cast<const float4*>(row + col));
                  v[q][0] = a4.x; v[q][1] = a4.y; v[q][2] = a4.z; v[q][3] = a4.w;
                }
                if (col + 4 < d) {
                  const float4 b4 = __ldg(reinterpret_cast<const float4*>(row + col + 4));
                  v[q][4] = b4.x; v[q][5] = b4.y; v[q][6] = b4.z; v[q][7] = b4.w;
                }
              }
            }
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = RPW * cw + 4 * (hb + q) + rsub;
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a = v[q][2 * k] * xs, b = v[q][2 * k + 1] * xs;
              const __half2 h = __floats2half2_rn(a, b);
              const float2 hf = __half22float2(h);
              const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
              hi[k] = *reinterpret_cast<const uint32_t*>(&h);
              lo[k] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const int off = r * 128 + ((c ^ (r & 7)) << 4);
            *reinterpret_cast<uint4*>(sa + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(sa + SM::A_BYTES + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
          __syncwarp();   // the second half's raw rows are read only after the first half's writes
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (TF32 && warp >= 12) {
    // ---- converters (TF32x2): the tile's points, fp32 -> hi = tf32_rn(x), lo = x - hi (exact in fp32; the MMA
    //      reads it as tf32, so |x - hi - lo| <= 2^-21 |x|), written in the 128-byte swizzled K-major layout:
    //      row r, 16-byte chunk c at r * 128 + ((c ^ (r % 8)) * 16).  Lane l: chunk l % 8 of rows 4 i + l / 8.
    const int cw = warp - 12;   // 0..3: rows 32 cw .. 32 cw + 31
    const int c = lane & 7, rsub = lane >> 3;
    if (xtma) {
      // the raw fp32 tile is the hi operand as it stands: kind::tf32 reads the top 19 bits of each 32-bit
      // container (truncation), so lo = x - trunc_tf32(x) completes it exactly in fp32
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t m0 = (t / ntn) * TC_M;
        const int split = (m0 < Nx && m0 + TC_M > Nx) ? static_cast<int>(Nx - m0) : TC_M;   // y rows >= split
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&xfull[stage], phase);
          unsigned char* sa = sm + stage * SM::STAGE;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = 32 * cw + 4 * it + rsub;
            const int off = r * 128 + ((c ^ (r & 7)) << 4);
            float4 v;
            if (r < split) {
              v = *reinterpret_cast<const float4*>(sa + off);
            } else {   // straddling tile: the y rows were loaded into the lo slot
              v = *reinterpret_cast<const float4*>(sa + SM::A_BYTES + off);
              *reinterpret_cast<float4*>(sa + off) = v;
            }
            const float4 lo = make_float4(tf32_cvt_rn(v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u)),
                                          tf32_cvt_rn(v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u)),
                                          tf32_cvt_rn(v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u)),
                                          tf32_cvt_rn(v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u)));
            *reinterpret_cast<float4*>(sa + SM::A_BYTES + off) = lo;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    } else {
    const bool vec = (d & 3) == 0;   // rows 16-byte aligned: one 16-byte load per chunk
    // software pipeline: the 8 chunks of the next (tile, k-block) are loaded into registers while the current
    // ones are converted and stored
    auto load8 = [&](int64_t m0, int kb, float4* v) {
      const int col = kb * 32 + 4 * c;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int64_t i = m0 + 32 * cw + 4 * it + rsub;
        v[it] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < L && col < d) {
          const float* row = (i < Nx) ? px + i * static_cast<int64_t>(d) : py + (i - Nx) * static_cast<int64_t>(d);
          if (vec) v[it] = __ldg(reinterpret_cast<const float4*>(row + col));
          else {
            v[it].x = __ldg(row + col);
            if (col + 1 < d) v[it].y = __ldg(row + col + 1);
            if (col + 2 < d) v[it].z = __ldg(row + col + 2);
            if (col + 3 < d) v[it].w = __ldg(row + col + 3);
          }
        }
      }
    };
    int stage = 0;
    uint32_t phase = 0;
    int64_t t = blockIdx.x;
    int kb = 0;
    float4 cur[8];
    if (t < ntiles) load8((t / ntn) * TC_M, 0, cur);
    while (t < ntiles) {
      // next (tile, k-block)
      int64_t tn = t;
      int kn = kb + 1;
      if (kn == nk) { kn = 0; tn += gridDim.x; }
      float4 nxt[8];
      if (tn < ntiles) load8((tn / ntn) * TC_M, kn, nxt);
      mbar_wait(&empty[stage], phase ^ 1);
      unsigned char* sa = sm + stage * SM::STAGE;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = 32 * cw + 4 * it + rsub;
        const float4 v = cur[it];
        const float4 hi = make_float4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
        const float4 lo = make_float4(tf32_cvt_rn(v.x - hi.x), tf32_cvt_rn(v.y - hi.y), tf32_cvt_rn(v.z - hi.z),
                                      tf32_cvt_rn(v.w - hi.w));
        const int off = r * 128 + ((c ^ (r & 7)) << 4);
        *reinterpret_cast<float4*>(sa + off) = hi;
        *reinterpret_cast<float4*>(sa + SM::A_BYTES + off) = lo;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
#pragma unroll
      for (int it = 0; it < 8; ++it) cur[it] = nxt[it];
      t = tn;
      kb = kn;
    }
    }
  } else if (warp >= 4 && warp < 4 + NEPI) {
    // ---- epilogue: warp w handles TMEM lane quadrant q = w % 4 (points m0 + 32q + lane) and the column part
    //      h = (w - 4) / 4 of the accumulator (two halves; FP16x2: all columns).  Per 16-column chunk: scale,
    //      store (coalesced along points), and the per-column min / max over the warp's 32 points by warp
    //      reductions (colrange16r).
    const int q = warp & 3, h = (warp - 4) >> 2;
    constexpr int HALF = BN / (NEPI / 4);
    float trap = 0.f;   // becomes NaN if a projection is NaN / Inf (in x, y or an overflow)
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      const uint32_t tph = (it >> 1) & 1;
      const int64_t m0 = (t / ntn) * TC_M;
      const int n0 = static_cast<int>(t % ntn) * BN + h * HALF;
      const int64_t w0 = m0 + 32 * q;
      const int64_t i = w0 + lane;
      const bool valid = i < L, isx = i < Nx;
      const bool warp_any_x = (w0 < Nx), mixed = warp_any_x && (w0 + 32 > Nx), warp_full = (w0 + 32 <= L);
      const int ncols = min(HALF, np - n0);   // may be <= 0
      mbar_wait(&tfull[b], tph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tbase =
          tmem_base + static_cast<uint32_t>(b * BN + h * HALF) + (static_cast<uint32_t>(32 * q) << 16);
      uint32_t v[16];
      if (ncols > 0)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tbase));
      float* zrow = Z + static_cast<int64_t>(n0) * ldz + i;
#pragma unroll 1
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t cur[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) cur[j] = v[j];
        if (c0 + 16 < ncols)   // prefetch the next 16 columns while this chunk is processed
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tbase + static_cast<uint32_t>(c0 + 16)));
        const int nc = min(16, ncols - c0);
        const float4* sv = reinterpret_cast<const float4*>(sinv + n0 + c0);
        float sc[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 f = sv[k];
          sc[4 * k] = f.x; sc[4 * k + 1] = f.y; sc[4 * k + 2] = f.z; sc[4 * k + 3] = f.w;
        }
        // scale + store (running pointer along the slices) + NaN/Inf trap; ranges as floats.  Full chunks (all
        // lanes valid, 16 columns) take a branch-free path.
        float fmn[16], fmx[16];
        float* zp = zrow + static_cast<int64_t>(c0) * ldz;
        if (warp_full && nc == 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            *zp = z;
            zp += ldz;
            trap = fmaf(z, 0.f, trap);   // NaN / Inf -> NaN
            fmn[j] = z;
            fmx[j] = z;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            const bool ok = valid && j < nc;
            if (ok) {
              *zp = z;
              trap = fmaf(z, 0.f, trap);
            }
            zp += ldz;
            fmn[j] = ok ? z : CUDART_INF_F;
            fmx[j] = ok ? z : -CUDART_INF_F;
          }
        }
        // per-column min / max over the warp's 32 points: one warp reduction per column and bound (redux.sync
        // f32, sm_100a), lane j keeps column j
        float amn, amx;
        colrange16r(fmn, fmx, lane, &amn, &amx);
        float xmn = amn, xmx = amx;
        if (mixed) {   // the warp holding the x/y boundary: x-only ranges separately
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            const bool ok = valid && isx && j < nc;
            fmn[j] = ok ? z : CUDART_INF_F;
            fmx[j] = ok ? z : -CUDART_INF_F;
          }
          colrange16r(fmn, fmx, lane, &xmn, &xmx);
        }
        if (lane < nc) {
          const int s = n0 + c0 + lane;
          if (amn <= amx) { atomicMin(&rng[4 * s + 2], f2key_tc(amn)); atomicMax(&rng[4 * s + 3], f2key_tc(amx)); }
          if (warp_any_x && xmn <= xmx) {
            atomicMin(&rng[4 * s + 0], f2key_tc(xmn));
            atomicMax(&rng[4 * s + 1], f2key_tc(xmx));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    if (__any_sync(0xffffffffu, trap != 0.f) && lane == 0) atomicOr(flag, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // this CTA's per-slice ranges into the global ranges (one atomic per slice and bound it touched); each CTA
  // starts at a different slice so that the CTAs finishing together do not queue on the same addresses
  const int ne = 4 * np, e0 = static_cast<int>((static_cast<int64_t>(blockIdx.x) * 4 * 61) % ne);
  for (int k = threadIdx.x; k < ne; k += blockDim.x) {
    const int e = (e0 + k) % ne;
    const unsigned v = rng[e];
    if ((e & 1) == 0) {
      if (v != 0xffffffffu) atomicMin(mm + e, v);
    } else if (v != 0u) {
      atomicMax(mm + e, v);
    }
  }
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
}

// ------------------------------------------------------------------ FP16x2 on CTA pairs (cta_group::2)
// The FP16x2 projection is bound by the SM's shared-memory pipe (TMA writes, converters, MMA operand reads: 224 KB
// per 64-dim k-block against 1024 tensor cycles).  A CTA pair (cluster of 2 on one TPC) computes a 256-point x
// 256-slice tile with tcgen05.mma.cta_group::2 (M = 256, N = 256): each CTA converts its own 128 points and
// loads only its half of the direction tile; the pair's tensor cores share the B halves, so each SM's shared
// memory serves half the direction bytes (176 KB per k-block).  Each CTA's TMEM holds its 128 points x 256 slices
// (double-buffered); the epilogue is the single-CTA one.  Barriers: per CTA xfull (raw tile landed), ready
// (converters done + own direction half landed), empty (MMA done, multicast commit to both CTAs), tfull (multicast);
// in the leader (rank 0) only: peer[stage] (the peer's ready, forwarded by its otherwise idle MMA warp with a
// cluster-scope arrive) and tempty (both CTAs' epilogue warps, count 2 NEPI).
constexpr int PR_STAGES = 4;
constexpr int PR_BN = 256;
constexpr int PR_A = TC_M * 128;          // one fp16 piece of 128 points x 64 dims (or a raw fp32 box of 32 dims)
constexpr int PR_BH = 128 * 128;          // this CTA's half of the direction tile: 128 slices x 64 dims
constexpr int PR_STAGE = 2 * PR_A + PR_BH;
constexpr int PR_BAR_OFF = PR_STAGES * PR_STAGE;
constexpr int PR_RANGE_OFF = (PR_BAR_OFF + 8 * (5 * PR_STAGES + 4) + 16 + 63) / 64 * 64;
constexpr int PR_FIXED = PR_RANGE_OFF + 1024;
constexpr int PR_NEPI = 4, PR_CW0 = 8, PR_NCONV = 8, PR_RPW = TC_M / PR_NCONV;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS_TF32, 1)
    k_proj_pair(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmY, int nk, int64_t L, int64_t Nx, int np,
                const float* __restrict__ inv_norm, float* __restrict__ Z, int64_t ldz, unsigned* __restrict__ mm,
                int* __restrict__ flag, const float* __restrict__ py, int d, const unsigned* __restrict__ f16max) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sm + PR_BAR_OFF);
  uint64_t* ready = xfull + PR_STAGES;
  uint64_t* peer = ready + PR_STAGES;
  uint64_t* empty = peer + PR_STAGES;
  uint64_t* tfull = empty + PR_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  unsigned* rng = reinterpret_cast<unsigned*>(sm + PR_RANGE_OFF);
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ntn = (np + PR_BN - 1) / PR_BN;
  float* sinv = reinterpret_cast<float*>(rng + 4 * ntn * PR_BN);
  const float zs = 1.0f / (256.0f * f16_scale(__ldg(f16max)));
  for (int c = threadIdx.x; c < ntn * PR_BN; c += blockDim.x) sinv[c] = (c < np) ? inv_norm[c] * zs : 0.f;
  const int64_t ntm = (L + 2 * TC_M - 1) / (2 * TC_M);
  const int64_t ntiles = ntm * ntn;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  for (int c = threadIdx.x; c < ntn * PR_BN; c += blockDim.x) {
    rng[4 * c + 0] = 0xffffffffu; rng[4 * c + 1] = 0u; rng[4 * c + 2] = 0xffffffffu; rng[4 * c + 3] = 0u;
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < PR_STAGES; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&ready[s], PR_NCONV + 1);
      mbar_init(&peer[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * PR_NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmY)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * PR_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();   // both CTAs' barriers initialised before any cross-CTA arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: this CTA's 128 raw fp32 points (two boxes of 32 dims) and its half of the direction tile
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = pair; t < ntiles; t += npairs) {
      const int64_t m0 = (t / ntn) * (2 * TC_M) + TC_M * rank;
      const int nb = static_cast<int>(t % ntn) * PR_BN + 128 * static_cast<int>(rank);
      const bool hasx = m0 < Nx;
      const CUtensorMap* mp = hasx ? &tmX : &tmY;
      const int row = hasx ? static_cast<int>(m0) : static_cast<int>(m0 - Nx);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* sa = sm + stage * PR_STAGE;
        mbar_expect_tx(&xfull[stage], 2 * PR_A);
        tma_load_2d(mp, &xfull[stage], sa, kb * 64, row);
        tma_load_2d(mp, &xfull[stage], sa + PR_A, kb * 64 + 32, row);
        mbar_expect_tx(&ready[stage], PR_BH);
        tma_load_2d(&tmB, &ready[stage], sa + 2 * PR_A, kb * TC_BK, nb);
        if (++stage == PR_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    if (leader) {
      // ---- MMA issuer (leader): D[256 points][256 slices] across the pair, K = 16 per MMA
      constexpr uint32_t idesc = idesc_f16(2 * TC_M, PR_BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t t = pair; t < ntiles; t += npairs, ++it) {
        const int b = it & 1;
        mbar_wait_cluster(&tempty[b], ((it >> 1) & 1) ^ 1);   // both CTAs' epilogues drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(b * PR_BN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&ready[stage], phase);
          mbar_wait_cluster(&peer[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const unsigned char* sa = sm + stage * PR_STAGE;
          const uint64_t db = umma_desc_sw128(sa + 2 * PR_A);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint64_t da = umma_desc_sw128(sa + q * PR_A);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t acc = (kb > 0 || q > 0 || k > 0) ? 1u : 0u;
              const uint64_t adv = static_cast<uint64_t>((k * 32) >> 4);
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                  "l"(da + adv), "l"(db + adv), "r"(idesc), "r"(acc));
            }
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[stage])),
              "h"(static_cast<uint16_t>(3))
              : "memory");
          if (++stage == PR_STAGES) { stage = 0; phase ^= 1; }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&tfull[b])),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      }
    } else {
      // ---- forwarder (peer): this CTA's stage is ready (its points converted, its direction half landed)
      const uint32_t rpeer = mapa_rank(&peer[0], 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = pair; t < ntiles; t += npairs)
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&ready[stage], phase);
          mbar_arrive_remote(rpeer + 8u * static_cast<uint32_t>(stage));
          if (++stage == PR_STAGES) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp >= PR_CW0) {
    // ---- converters (as k_proj_tc MODE 3): the raw fp32 rows of a k-block -> fp16 hi / lo of the scaled points
    const int cw = warp - PR_CW0;
    const int c = lane & 7, rsub = lane >> 3;
    const float xs = f16_scale(__ldg(f16max));
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = pair; t < ntiles; t += npairs) {
      const int64_t m0 = (t / ntn) * (2 * TC_M) + TC_M * rank;
      const int split = (m0 < Nx && m0 + TC_M > Nx) ? static_cast<int>(Nx - m0) : TC_M;   // y rows >= split
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&xfull[stage], phase);
        unsigned char* sa = sm + stage * PR_STAGE;
        float v[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = PR_RPW * cw + 4 * q + rsub;
          const int box = c >> 2, j0 = 2 * (c & 3);
          const unsigned char* rb = sa + box * PR_A + r * 128;
          if (r < split) {
            const int jf = j0 + box, js = j0 + 1 - box;
            const float4 f4 = *reinterpret_cast<const float4*>(rb + ((jf ^ (r & 7)) << 4));
            const float4 s4 = *reinterpret_cast<const float4*>(rb + ((js ^ (r & 7)) << 4));
            const float4 a4 = box ? s4 : f4, b4 = box ? f4 : s4;
            v[q][0] = a4.x; v[q][1] = a4.y; v[q][2] = a4.z; v[q][3] = a4.w;
            v[q][4] = b4.x; v[q][5] = b4.y; v[q][6] = b4.z; v[q][7] = b4.w;
          } else {   // straddling tile: y rows from global memory
            const int64_t i = m0 + r;
            const int col = kb * 64 + 8 * c;
#pragma unroll
            for (int u = 0; u < 8; ++u) v[q][u] = 0.f;
            if (i < L) {
              const float* rowp = py + (i - Nx) * static_cast<int64_t>(d);
              if (col < d) {
                const float4 a4 = __ldg(reinterpret_cast<const float4*>(rowp + col));
                v[q][0] = a4.x; v[q][1] = a4.y; v[q][2] = a4.z; v[q][3] = a4.w;
              }
              if (col + 4 < d) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(rowp + col + 4));
                v[q][4] = b4.x; v[q][5] = b4.y; v[q][6] = b4.z; v[q][7] = b4.w;
              }
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = PR_RPW * cw + 4 * q + rsub;
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float a = v[q][2 * k] * xs, b = v[q][2 * k + 1] * xs;
            const __half2 h = __floats2half2_rn(a, b);
            const float2 hf = __half22float2(h);
            const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
            hi[k] = *reinterpret_cast<const uint32_t*>(&h);
            lo[k] = *reinterpret_cast<const uint32_t*>(&l);
          }
          const int off = r * 128 + ((c ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(sa + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(sa + PR_A + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[stage]);
        if (++stage == PR_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 4 + PR_NEPI) {
    // ---- epilogue (as k_proj_tc): warp w, TMEM lane quadrant q = w % 4 of this CTA's 128 points, all 256 slices
    const int q = warp & 3;
    const uint32_t rtempty = mapa_rank(&tempty[0], 0);
    float trap = 0.f;
    int it = 0;
    for (int64_t t = pair; t < ntiles; t += npairs, ++it) {
      const int b = it & 1;
      const uint32_t tph = (it >> 1) & 1;
      const int64_t m0 = (t / ntn) * (2 * TC_M) + TC_M * rank;
      const int n0 = static_cast<int>(t % ntn) * PR_BN;
      const int64_t w0 = m0 + 32 * q;
      const int64_t i = w0 + lane;
      const bool valid = i < L, isx = i < Nx;
      const bool warp_any_x = (w0 < Nx), mixed = warp_any_x && (w0 + 32 > Nx), warp_full = (w0 + 32 <= L);
      const int ncols = min(PR_BN, np - n0);
      mbar_wait(&tfull[b], tph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tbase = tmem_base + static_cast<uint32_t>(b * PR_BN) + (static_cast<uint32_t>(32 * q) << 16);
      uint32_t v[16];
      if (ncols > 0)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tbase));
      float* zrow = Z + static_cast<int64_t>(n0) * ldz + i;
#pragma unroll 1
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t cur[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) cur[j] = v[j];
        if (c0 + 16 < ncols)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tbase + static_cast<uint32_t>(c0 + 16)));
        const int nc = min(16, ncols - c0);
        const float4* sv = reinterpret_cast<const float4*>(sinv + n0 + c0);
        float sc[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 f = sv[k];
          sc[4 * k] = f.x; sc[4 * k + 1] = f.y; sc[4 * k + 2] = f.z; sc[4 * k + 3] = f.w;
        }
        float fmn[16], fmx[16];
        float* zp = zrow + static_cast<int64_t>(c0) * ldz;
        if (warp_full && nc == 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            *zp = z;
            zp += ldz;
            trap = fmaf(z, 0.f, trap);
            fmn[j] = z;
            fmx[j] = z;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            const bool ok = valid && j < nc;
            if (ok) {
              *zp = z;
              trap = fmaf(z, 0.f, trap);
            }
            zp += ldz;
            fmn[j] = ok ? z : CUDART_INF_F;
            fmx[j] = ok ? z : -CUDART_INF_F;
          }
        }
        float amn, amx;
        colrange16r(fmn, fmx, lane, &amn, &amx);
        float xmn = amn, xmx = amx;
        if (mixed) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(cur[j]) * sc[j];
            const bool ok = valid && isx && j < nc;
            fmn[j] = ok ? z : CUDART_INF_F;
            fmx[j] = ok ? z : -CUDART_INF_F;
          }
          colrange16r(fmn, fmx, lane, &xmn, &xmx);
        }
        if (lane < nc) {
          const int s = n0 + c0 + lane;
          if (amn <= amx) { atomicMin(&rng[4 * s + 2], f2key_tc(amn)); atomicMax(&rng[4 * s + 3], f2key_tc(amx)); }
          if (warp_any_x && xmn <= xmx) {
            atomicMin(&rng[4 * s + 0], f2key_tc(xmn));
            atomicMax(&rng[4 * s + 1], f2key_tc(xmx));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {   // release the accumulator to the leader's MMA of tile t + 2 (both CTAs' epilogues)
        if (leader) mbar_arrive(&tempty[b]);
        else mbar_arrive_remote(rtempty + 8u * static_cast<uint32_t>(b));
      }
    }
    if (__any_sync(0xffffffffu, trap != 0.f) && lane == 0) atomicOr(flag, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();   // the peer's remote arrives and both CTAs' TMEM reads are done before the pair deallocates
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int ne = 4 * np, e0 = static_cast<int>((static_cast<int64_t>(blockIdx.x) * 4 * 61) % ne);
  for (int k = threadIdx.x; k < ne; k += blockDim.x) {
    const int e = (e0 + k) % ne;
    const unsigned v = rng[e];
    if ((e & 1) == 0) {
      if (v != 0xffffffffu) atomicMin(mm + e, v);
    } else if (v != 0u) {
      atomicMax(mm + e, v);
    }
  }
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * PR_BN));
}

// fp32 -> three bf16 pieces, K-concatenated:  Xs[i][j] = hi, Xs[i][dp+j] = mid, Xs[i][2dp+j] = lo.
// One thread per 8 consecutive coordinates of a row: vector loads when the row is 16-byte aligned,
// three 16-byte stores (dp is a multiple of 64, so every 8-group is aligned in Xs).
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& mid, uint4& lo) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat16 hh[2], mm[2], ll[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float x = v[2 * q + r];
      hh[r] = __float2bfloat16_rn(x);
      const float r1 = x - __bfloat162float(hh[r]);
      mm[r] = __float2bfloat16_rn(r1);
      ll[r] = __float2bfloat16_rn(r1 - __bfloat162float(mm[r]));
    }
    h[q] = static_cast<uint32_t>(__bfloat16_as_ushort(hh[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(hh[1])) << 16);
    m[q] = static_cast<uint32_t>(__bfloat16_as_ushort(mm[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(mm[1])) << 16);
    l[q] = static_cast<uint32_t>(__bfloat16_as_ushort(ll[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(ll[1])) << 16);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  mid = make_uint4(m[0], m[1], m[2], m[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void k_split3(const float* __restrict__ x, int64_t N, const float* __restrict__ y, int64_t M, int d, int dp,
                         __nv_bfloat16* __restrict__ xs) {
  const int64_t L = N + M;
  const int g8 = dp / 8;   // 8-groups per row
  const int64_t total = L * g8;
  const bool vec = (d % 4) == 0;   // rows 16-byte aligned (base pointers from cudaMalloc/torch are 256-aligned)
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / g8;
    const int j0 = static_cast<int>(e - i * g8) * 8;
    const float* row = (i < N) ? x + i * d : y + (i - N) * d;
    float v[8];
    if (vec && j0 + 8 <= d) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(row + j0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(row + j0 + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (j0 + u < d) ? __ldg(row + j0 + u) : 0.f;
    }
    uint4 hi, mid, lo;
    split8(v, hi, mid, lo);
    uint4* out = reinterpret_cast<uint4*>(xs + i * (3 * static_cast<int64_t>(dp)) + j0);
    out[0] = hi;
    out[dp / 8] = mid;
    out[2 * (dp / 8)] = lo;
  }
}

bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols_k, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {cols_k, rows};
  const cuuint64_t gstride[1] = {cols_k * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(TC_BK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int STAGES, int MODE = 0>
cudaError_t launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, int nk, int64_t L, int64_t Nx, int np,
                      const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag, unsigned* part,
                      cudaStream_t st, const float* px = nullptr, const float* py = nullptr, int d = 0,
                      const CUtensorMap* tx = nullptr, const CUtensorMap* ty = nullptr,
                      const unsigned* f16max = nullptr, const unsigned* pred = nullptr) {
  using SM = TcSmem<BN, STAGES, MODE>;
  const int ntn = (np + BN - 1) / BN;
  const size_t smem = SM::FIXED + static_cast<size_t>(20) * ntn * BN;
  set_smem_attr_once(reinterpret_cast<const void*>(k_proj_tc<BN, STAGES, MODE>), 227 * 1024);
  const int64_t ntiles = ((L + TC_M - 1) / TC_M) * ntn;
  const int grid = static_cast<int>(ntiles < kProjMaxCtas ? ntiles : kProjMaxCtas);
  const int xtma = tx != nullptr;
  k_proj_tc<BN, STAGES, MODE><<<grid, MODE != 0 ? TC_THREADS_TF32 : TC_THREADS, smem, st>>>(
      ta, tb, nk, L, Nx, np, inv_norm, Z, ldz, mm, flag, px, py, d, xtma ? *tx : ta, xtma ? *ty : ta, xtma,
      f16max, pred);
  (void)part;
  return cudaGetLastError();
}

// direction tile of the TF32x2 path: fp32 [np][dp32] (values bf16-exact, hence tf32-exact), box 32 x rows
bool make_map_f32(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {cols * 4};
  const cuuint32_t box[2] = {32, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// raw fp32 points [rows][d] for the TF32x2 path: box 32 dims x 128 rows, 128-byte swizzle (the hi operand layout);
// dims >= d and rows outside [0, rows) are zero-filled
bool make_map_pts(CUtensorMap* m, const float* base, uint64_t rows, uint64_t d) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {d, rows};
  const cuuint64_t gstride[1] = {d * 4};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(TC_M)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int proj_tc_dpad(int d) { return (d + TC_BK - 1) / TC_BK * TC_BK; }

bool proj_tf32_tma_ok(const float* x, int64_t N, const float* y, int64_t M, int d) {
  return (d % 4) == 0 && N > 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0 &&
         (M == 0 || (reinterpret_cast<uintptr_t>(y) % 16) == 0);
}
int proj_tf32_dpad(int d) { return (d + 31) / 32 * 32; }

// Z = X G^T with the TF32x2 split done inside the kernel (converter warps read the fp32 points directly):
// no split buffer; three k-blocks of 32 dims per 128-byte row pair... see k_proj_tc<.., true>
cudaError_t launch_project_tf32(const float* x, int64_t N, const float* y, int64_t M, int d,
                                const float* g32 /* fp32 [np][dp32] */, int np, const float* inv_norm, float* Z,
                                int64_t ldz, unsigned* mm, int* flag, const unsigned* pred, cudaStream_t st) {
  const int dp = proj_tf32_dpad(d);
  const int nk = dp / 32;
  const int64_t L = N + M;
  CUtensorMap ta;
  std::memset(&ta, 0, sizeof(ta));   // unused by the TF32 path
  // raw points by TMA (fp32 rows of d floats, box 32 dims x 128 rows, 128-byte swizzle): needs 16-byte row
  // strides and bases; otherwise the converter warps load them
  CUtensorMap tx, ty;
  bool xtma = proj_tf32_tma_ok(x, N, y, M, d);
  if (xtma) {
    xtma = make_map_pts(&tx, x, static_cast<uint64_t>(N), static_cast<uint64_t>(d)) &&
           (M == 0 ? (ty = tx, true) : make_map_pts(&ty, y, static_cast<uint64_t>(M), static_cast<uint64_t>(d)));
  }
  const CUtensorMap* ptx = xtma ? &tx : nullptr;
  const CUtensorMap* pty = xtma ? &ty : nullptr;
  constexpr int kSliceChunk = 1024;
  for (int s0 = 0; s0 < np; s0 += kSliceChunk) {
    const int ns = std::min(kSliceChunk, np - s0);
    const int BN = ns > 128 ? 256 : (ns > 64 ? 128 : 64);
    CUtensorMap tb;
    if (!make_map_f32(&tb, g32 + static_cast<int64_t>(s0) * dp, static_cast<uint64_t>(ns), static_cast<uint64_t>(dp),
                      static_cast<uint32_t>(BN)))
      return cudaErrorInvalidValue;
    float* Zc = Z + static_cast<int64_t>(s0) * ldz;
    unsigned* mmc = mm + 4 * s0;
    const float* ic = inv_norm + s0;
    cudaError_t e;
    if (BN == 256) e = launch_tc<256, 3, 1>(ta, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, ptx, pty, nullptr, pred);
    else if (BN == 128) e = launch_tc<128, 4, 1>(ta, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, ptx, pty, nullptr, pred);
    else e = launch_tc<64, 4, 1>(ta, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, ptx, pty, nullptr, pred);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// FP16x2 (MODE 3): points by TMA (needs proj_tf32_tma_ok), directions g16 = fp16(2^8 g) [np][dp] (dp = 64-padded);
// f16max: 4 zeroed bytes of scratch for the sampled max |x|; a point with |s x| >= 2^15 sets flag bit 1
cudaError_t launch_project_f16(const float* x, int64_t N, const float* y, int64_t M, int d, const void* g16, int np,
                               const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag,
                               unsigned* f16max, cudaStream_t st) {
  const int dp = proj_tc_dpad(d);
  const int nk = dp / TC_BK;
  const int64_t L = N + M;
  CUtensorMap tx, ty;
  if (!make_map_pts(&tx, x, static_cast<uint64_t>(N), static_cast<uint64_t>(d))) return cudaErrorInvalidValue;
  if (M == 0) ty = tx;
  else if (!make_map_pts(&ty, y, static_cast<uint64_t>(M), static_cast<uint64_t>(d))) return cudaErrorInvalidValue;
  const int S = static_cast<int>(std::min<int64_t>(L, 1024));
  k_absmax_sample<<<S, 256, 0, st>>>(x, N, y, M, d, S, f16max);
  constexpr int kSliceChunk = 1024;
  for (int s0 = 0; s0 < np; s0 += kSliceChunk) {
    const int ns = std::min(kSliceChunk, np - s0);
    const int BN = ns > 128 ? 256 : (ns > 64 ? 128 : 64);
    const void* g = static_cast<const uint16_t*>(g16) + static_cast<int64_t>(s0) * dp;
    CUtensorMap tb;
    if (!make_map(&tb, g, static_cast<uint64_t>(ns), static_cast<uint64_t>(dp), static_cast<uint32_t>(BN)))
      return cudaErrorInvalidValue;
    float* Zc = Z + static_cast<int64_t>(s0) * ldz;
    unsigned* mmc = mm + 4 * s0;
    const float* ic = inv_norm + s0;
    cudaError_t e;
    if (BN == 256 && L >= 2 * TC_M) {   // CTA pairs (cta_group::2): half the direction bytes per SM
      CUtensorMap th;
      if (!make_map(&th, g, static_cast<uint64_t>(ns), static_cast<uint64_t>(dp), 128u)) return cudaErrorInvalidValue;
      const int ntn = (ns + PR_BN - 1) / PR_BN;
      const size_t smem = PR_FIXED + static_cast<size_t>(20) * ntn * PR_BN;
      set_smem_attr_once(reinterpret_cast<const void*>(k_proj_pair), 227 * 1024);
      const int64_t ntiles = ((L + 2 * TC_M - 1) / (2 * TC_M)) * ntn;
      const int pairs = static_cast<int>(ntiles < kProjMaxCtas / 2 ? ntiles : kProjMaxCtas / 2);
      k_proj_pair<<<2 * pairs, TC_THREADS_TF32, smem, st>>>(th, tx, ty, nk, L, N, ns, ic, Zc, ldz, mmc, flag, y, d,
                                                            f16max);
      e = cudaGetLastError();
    } else if (BN == 256) e = launch_tc<256, 3, 3>(tb, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, &tx, &ty, f16max);
    else if (BN == 128) e = launch_tc<128, 4, 3>(tb, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, &tx, &ty, f16max);
    else e = launch_tc<64, 4, 3>(tb, tb, nk, L, N, ns, ic, Zc, ldz, mmc, flag, nullptr, st, x, y, d, &tx, &ty, f16max);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_split3(const float* x, int64_t N, const float* y, int64_t M, int d, void* xs, cudaStream_t st) {
  const int dp = proj_tc_dpad(d);
  const int64_t total = (N + M) * (dp / 8);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_split3<<<static_cast<unsigned>(blocks), 256, 0, st>>>(x, N, y, M, d, dp, static_cast<__nv_bfloat16*>(xs));
  return cudaGetLastError();
}

size_t proj_tc_part_bytes(int np) { return static_cast<size_t>(kProjMaxCtas) * 16 * np; }

cudaError_t launch_project_tc(const void* xs, int64_t L, int64_t Nx, int d, const void* g3 /* bf16 [np][dp] */, int np,
                              const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag, void* part,
                              cudaStream_t st) {
  const int dp = proj_tc_dpad(d);
  const int nk = dp / TC_BK;
  CUtensorMap ta;
  if (!make_map(&ta, xs, static_cast<uint64_t>(L), static_cast<uint64_t>(3 * dp), TC_M)) return cudaErrorInvalidValue;
  unsigned* pp = static_cast<unsigned*>(part);
  // the per-CTA range partials of all its slices live in shared memory (20 B per slice): launches of at most
  // kSliceChunk slices (the point tiles are re-read per launch, from L2 for moderate L)
  constexpr int kSliceChunk = 1024;
  for (int s0 = 0; s0 < np; s0 += kSliceChunk) {
    const int ns = std::min(kSliceChunk, np - s0);
    const int BN = ns > 128 ? 256 : (ns > 64 ? 128 : 64);
    const void* g = static_cast<const uint16_t*>(g3) + static_cast<int64_t>(s0) * dp;
    CUtensorMap tb;
    if (!make_map(&tb, g, static_cast<uint64_t>(ns), static_cast<uint64_t>(dp), static_cast<uint32_t>(BN)))
      return cudaErrorInvalidValue;
    float* Zc = Z + static_cast<int64_t>(s0) * ldz;
    unsigned* mmc = mm + 4 * s0;
    const float* ic = inv_norm + s0;
    cudaError_t e;
    if (BN == 256) e = launch_tc<256, 2>(ta, tb, nk, L, Nx, ns, ic, Zc, ldz, mmc, flag, pp, st);
    else if (BN == 128) e = launch_tc<128, 3>(ta, tb, nk, L, Nx, ns, ic, Zc, ldz, mmc, flag, pp, st);
    else e = launch_tc<64, 3>(ta, tb, nk, L, Nx, ns, ic, Zc, ldz, mmc, flag, pp, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sks
