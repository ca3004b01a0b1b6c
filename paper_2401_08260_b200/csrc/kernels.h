// kernels.h -- launch wrappers of the sm_100a kernels of libsks (defined in *.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

// Checked builds (-DSKS_CHECKS, build.py --checked -> libsks_checked.so): device-side bounds checks on every data-
// dependent index (grid cells, polynomial tables, mailbox slots, sort ranks) that trap with a message.  They stand in
// for compute-sanitizer, which this pool does not run; tests/test_checked_build.py drives every kernel through them.
#if defined(SKS_CHECKS) && defined(__CUDACC__)
#include <cstdio>
#define SKS_CHECK(c)                                                                          \
  do {                                                                                        \
    if (!(c)) {                                                                               \
      printf("SKS_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,           \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x), #c);                 \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define SKS_CHECK(c) \
  do {               \
  } while (0)
#endif

namespace sks {

// opt-in per-launch timing (sks_profile_*, api.cpp): CUDA events around launches, accumulated per slot
enum ProfSlot {
  PS_SPLIT = 0, PS_PROJECT, PS_MINMAX, PS_SP_HIST, PS_SP_PART, PS_SP_OWNER, PS_SP_GATHER, PS_RESERVED, PS_PLAN,
  PS_SPREAD, PS_FFT, PS_EVAL, PS_AUX, PS_NDFT_SPREAD, PS_NDFT_EVAL, PS_SORT, PS_N
};
struct ProfMark {
  int slot;
  cudaStream_t st;
  cudaEvent_t a;   // nullptr when profiling is off
};
ProfMark prof_begin(int slot, cudaStream_t st);
void prof_end(const ProfMark& m);

// raise a kernel's dynamic shared-memory limit to `bytes` on the current device (function attributes are per
// device): set once per (kernel, device), thread-safe
void set_smem_attr_once(const void* kernel, int bytes);

// per-slice Fourier plan (row a2), written by the device planner k_plan (plan.cu)
struct FPar {
  float tau, cen;   // u = tau (z - cen)
  int lmin;         // first cell of the x footprint (spreading)
  int klo, khi;     // kept band klo <= |k| <= khi
  int lminA;        // first cell of the all-points footprint (interpolation polynomials)
  int logn;         // grid n = 2^logn
  int W, WA;        // widths (cells) of the x / all-points footprints
  int pad[3];
};

// flag words of a call (16 bytes in the workspace): [0] non-finite projection, [1] FP16x2 sampled max |x|,
// [2] plan failure bits (1: grid beyond n_cap, 2: band too wide for the NDFT), [3] FP16x2 range exceeded (the
// projection was redone on TF32x2).  Kernels after the planner exit at once if [0] or [2] is set.
__device__ __forceinline__ bool call_failed(const unsigned* flag16) { return (flag16[0] | flag16[2]) != 0; }

// window polynomials: tap j weight p_j(f) = sum_k c[j*(PW_D+1)+k] f^k, f = frac(v - w/2)  (R6)
constexpr int PW_D = 7;   // == host kPolyDeg; 8 coefficients = two float4
struct PolyWin {
  int w;
  float c[12 * (PW_D + 1)];
  // centered form for spreading: with u = f - 1/2, tap j < w/2 has p_j = E_j(u^2) + u O_j(u^2) and the mirror tap
  // p_{w-1-j}(f) := p_j(1 - f) = E_j(u^2) - u O_j(u^2)  (the ES window is even); eo[j] = {E_j[0..3], O_j[0..3]}
  float eo[6][8];
};

// per-call constants of the closed-form torus coefficients (device planner, row a2)
struct CoeffConst {
  int kind, d;
  double scale;     // sigma | ell | beta
  double logpref;   // log of the constant prefactor of fhat1 (see host: fhat1)
  double nu;        // Matern nu
  double lap_A;     // Laplacian: c_d / scale  (alpha c_d), multiplied by 1/tau per slice
};

// data-independent inputs of the device planner (host, cached per (kernel, d, eps, w, os))
struct PlanConst {
  CoeffConst cc;
  double reps;      // decay radius r_eps of the counterpart (x units, reading R3)
  double eps;       // dropped-coefficient budget (R5)
  int os, w;        // oversampling, window taps
  int ncap_log;     // log2 of the largest grid (n_cap)
  int ndft;         // 1: the NDFT engine (band <= 32, no window deconvolution)
};
constexpr int kPlanSummaryWords = 8;   // max n, max k_hi, min k_lo, max W, max band, tau min / max bits, max WA

// Where a kernel's per-(target, slice group) sums go: fp64 atomics into s64 (default), or -- deterministic mode
// (sks_options.deterministic) -- plain stores part[(goff + group) * M + m], added in a fixed order by
// launch_finalize_det.  Every (group, target) of a launch is written exactly once.
struct TargetAcc {
  double* s64;
  double* part;
  int64_t M;
  int goff;
};
#if defined(__CUDACC__)
__device__ __forceinline__ void acc_target(const TargetAcc& t, int grp, int64_t m, double v) {
  if (t.part) t.part[(static_cast<int64_t>(t.goff) + grp) * t.M + m] = v;
  else if (t.s64) atomicAdd(t.s64 + m, v);
}
#endif

// views of the projected points of a slice batch: x-part zx[p*ldx + i], y-part zy[p*ldy + m]
struct ZView {
  const float* zx;
  const float* zy;
  int64_t ldx, ldy;
  int64_t N, M;
};

// row a1 (proj_tc.cu): Z[p][i] = inv_norm[p] * <g_p, pt_i>, i in [0, N+M) (x block then y block); per-slice ranges
// mm[p*4 + {0,1,2,3}] = encoded {xmin, xmax, allmin, allmax}; non-finite flag.
// row a1 on tensor cores (proj_tc.cu): split fp32 points into 3 bf16 pieces (K-concatenated, d padded to
// dp = proj_tc_dpad(d)), then Z = Xs . G3^T on tcgen05 with TMA/TMEM, same epilogue contract as above.
int proj_tc_dpad(int d);
cudaError_t launch_split3(const float* x, int64_t N, const float* y, int64_t M, int d, void* xs, cudaStream_t st);
size_t proj_tc_part_bytes(int np);   // scratch for per-CTA range partials
cudaError_t launch_project_tc(const void* xs, int64_t L, int64_t Nx, int d, const void* g3, int np,
                              const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag, void* part,
                              cudaStream_t st);
// row a1 as TF32x2 with the split inside the kernel (small d: no split buffer, the fp32 points are read once):
// hi = tf32_rn(x), lo = x - hi, two kind::tf32 MMAs against the fp32 (tf32-exact) directions g32 [np][dp32]
int proj_tf32_dpad(int d);
// row a1 as FP16x2: s x = hi + lo in fp16 (s = 2^e from a sampled max |x|), directions as fp16(2^8 g), two
// kind::f16 MMAs (twice the tf32 rate, the precision of TF32x2).  Needs proj_tf32_tma_ok; f16max = 4 zeroed
// scratch bytes; flag bit 1 = a point outside the fp16 range (rerun with TF32x2)
cudaError_t launch_project_f16(const float* x, int64_t N, const float* y, int64_t M, int d, const void* g16, int np,
                               const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag,
                               unsigned* f16max, cudaStream_t st);
// the points can be read by TMA (d % 4 == 0, 16-byte aligned arrays): the raw fp32 tile is the hi operand
bool proj_tf32_tma_ok(const float* x, int64_t N, const float* y, int64_t M, int d);
// pred: nullptr, or a device word; the launch does nothing unless *pred != 0 (the FP16x2 -> TF32x2 rerun)
cudaError_t launch_project_tf32(const float* x, int64_t N, const float* y, int64_t M, int d, const float* g32, int np,
                                const float* inv_norm, float* Z, int64_t ldz, unsigned* mm, int* flag,
                                const unsigned* pred, cudaStream_t st);
// after an FP16x2 projection: if it flagged a non-finite value (a point beyond the fp16 range, or a NaN / Inf input),
// move the flag to flag16[3] (rerun) and reset the ranges mm [np][4], so that the predicated TF32x2 launch redoes the
// batch (and flags genuine NaN / Inf inputs again)
cudaError_t launch_rerun_prep(unsigned* flag16, unsigned* mm, int np, cudaStream_t st);
// per-slice ranges of given projections (sks_sum_1d)
cudaError_t launch_minmax(ZView zv, int np, unsigned* mm, int* flag, cudaStream_t st);
cudaError_t launch_init_minmax(unsigned* mm, int np, cudaStream_t st);
// call prologue (one launch): flag16 (16 bytes) zeroed, the plan summary at flag16 + 16 bytes initialised, s64 [M]
// (nullptr: none) zeroed, mm [np][4] initialised
cudaError_t launch_prologue(void* flag16, double* s64, int64_t M, unsigned* mm, int np, cudaStream_t st);
void decode_minmax(const unsigned* enc, float* dec, int n);

struct SliceTot {
  double A, B, C, pad;   // sum w, sum w z, sum w z^2 over the slice's sources
};
// rows a3 + a4, owner-partitioned (sortpart.cu): histogram -> G owners per slice (contiguous value
// ranges balanced by x count) -> coalesced partition into per-owner mailboxes -> per-owner fine-bucket
// counting sort, fp64 prefix sums and target evaluation in shared memory -> gather back to target order.
struct SpOwner {         // one owner (contiguous bin range [blo, blo + NBF/fmul)) of one slice
  int xoff, xcnt;        // its x in the slice's x mailbox
  int yoff, ycnt;        // its y in the slice's y mailbox
  float blo, fmul;       // fine bucket = floor((u - blo) * fmul), u = bin coordinate
  int pad0, pad1;
};
struct SpDims {
  int NH = 0;            // histogram bins per slice
  int G = 0;             // owners per slice
};
struct SortPartArgs {
  ZView zv;
  const float* w;
  int np;
  const unsigned* mm;    // [np][4] ranges
  SliceTot* tot;         // [np] sum w, sum w z, sum w z^2 (fp64)
  double coef;           // t = -coef * sum_n w_n |x_n - z|
  TargetAcc acc;         // accumulate sum_p t per target (fp64; deterministic mode: one group per gather row), or
  float* per_slice_out;  // store t into per_slice_out[p*M + m]
  bool det;              // deterministic mode: each owner's buckets ordered by value before they are summed
};
SpDims sortpart_dims(int64_t N, int64_t M);
int sortpart_acc_groups(int64_t N, int64_t M, int np);   // TargetAcc groups one launch_sortpart writes
size_t sortpart_bytes(int64_t N, int64_t M, int np);   // scratch of launch_sortpart
int sortpart_group(int64_t N, int64_t M, int np);      // slices per L2-resident group
int sortpart_launches_per_group(int64_t N, int64_t M);   // kernels per group (4, or 5 with many owners)
inline int sortpart_groups(int64_t N, int64_t M, int np) {
  const int g = sortpart_group(N, M, np);
  return (np + g - 1) / g;
}
cudaError_t launch_sortpart(const SortPartArgs& a, void* ws, cudaStream_t st);

// row a2 (plan.cu): per slice, from the ranges mm [np][4]: FPar fp[p], D[p][k] (stride n_cap/2 + 1) =
// c_k(tau_p) / Phi(k / n_p)^2 on the band (phi2inv_cap[j] = 1 / Phi(j / n_cap)^2), grid[p][0, n_p) zeroed (stride
// n_cap); failures set flag16 bits; summary [kPlanSummaryWords] (initialised by the prologue)
cudaError_t launch_plan(const unsigned* mm, int np, const PlanConst& pc, const float* phi2inv_cap, FPar* fp, float* D,
                        float* grid, unsigned* flag16, unsigned* summary, cudaStream_t st);
// rows a1 + a5 fused (fused.cu; sources only, Fourier kernels at large N): the sources' projections are spread into
// the grids from the tensor-core accumulators, never stored.  fused_spread_ok: d <= 128, d % 4 == 0, 16-byte
// aligned x.  launch_source_prep, then per batch launch_bound_ranges (mu: source_bound_bytes(d) of scratch, nb: its
// last 32 bytes), launch_plan, launch_proj_spread in place of the projection of x + launch_spread
bool fused_spread_ok(int d, const float* x);
size_t source_bound_bytes(int d);   // scratch of launch_source_prep: mu, partial sums, nb (32 bytes, at the end)
// launch_source_prep (once per call, direction-independent): mu, the norm words nb (max ||z - mu||^2, max ||z||^2,
// non-finite) of x (nb[0..2]) and y (nb[4..6]), and both point sets as the fused kernels' FP16x2 operands in the
// same pass: per 8-row group g a scale s_g = 2^(14 - e) (max |z| over the group = m 2^e), hi = f16(s_g z),
// lo = f16(s_g z - hi) as fp16 arrays [rows][fused_dp16(d)] (pad columns zero), rs[g] = 1 / (2^8 s_g) (reading R2),
// and the source weights w zero padded to whole 128-point tiles (wpad, read by the spread's bulk copies).
// launch_bound_ranges (per slice batch): every slice's range bound c_p +- rho' of both sets into mm[p]
int fused_dp16(int d);   // row length of the fp16 operand arrays: d rounded up to 8
// launch_source_mean: mu (and nb zeroed), before launch_source_prep (between them a point-sharded call makes every
// rank adopt rank 0's mu; after it the ranks take the maxima of nb: sks.h sks_exchange_fn)
cudaError_t launch_source_mean(const float* x, int64_t N, int d, double* mu, unsigned* nb, cudaStream_t st);
cudaError_t launch_source_prep(const float* x, int64_t N, const float* y, int64_t M, int d, const double* mu,
                               unsigned* nb, uint16_t* xh, uint16_t* xl, float* rsx, uint16_t* yh, uint16_t* yl,
                               float* rsy, const float* w, float* wpad, cudaStream_t st);
cudaError_t launch_bound_ranges(const float* g32, int dp32, int d, const float* inv_norm, int np, const double* mu,
                                const unsigned* nb, unsigned* mm, unsigned* flag16, cudaStream_t st);
// g16: the slices' fp16 directions 2^8 g, row stride dpg (a multiple of 64)
cudaError_t launch_proj_spread(const uint16_t* xh, const uint16_t* xl, const float* rsx, int64_t N, int d,
                               const uint16_t* g16, int dpg, const float* inv_norm, int np, const float* wpad,
                               const FPar* fp, const PolyWin& pw, int ncap, float* grid, const unsigned* flag16,
                               cudaStream_t st);
// rows a1 + a7 fused for the targets (fused.cu): projections of y interpolated from the tensor-core accumulators,
// s64[m] += sum over the slices of t_{m,p} (after launch_fft_filter wrote Q)
cudaError_t launch_proj_eval(const uint16_t* yh, const uint16_t* yl, const float* rsy, int64_t M, int d,
                             const uint16_t* g16, int dpg, const float* inv_norm, int np, const FPar* fp,
                             const float* Q, int ncap, int w, double* s64, const unsigned* flag16, cudaStream_t st);
// row a5: g[p][l] = sum_n w_n phi_win(v_n - l) over the x projections (ES window, w taps); grid stride n_cap
// det: one CTA per slice (no cross-CTA grid accumulation; the private grids are reduced in a fixed order)
cudaError_t launch_spread(ZView zv, const float* w, int np, const FPar* fp, int ncap, const PolyWin& pw,
                          bool wide_likely, bool det, float* grid, const unsigned* flag16, cudaStream_t st);
// row a6: h[p] = IFFT_n(D[p] * FFT_n(g[p]))   (unnormalised, one CTA per slice, smem radix-2, n = n_p)
// also writes the per-cell interpolation polynomials Q[p][c][k] = sum_j h[lminA + c + j] coef[j][k] for the
// WA cells of the all-points footprint (Q stride kQStride(n_cap) floats per slice)
__host__ __device__ inline int64_t q_stride(int ncap) { return static_cast<int64_t>(ncap + 16) * (PW_D + 1); }
// (cap_hint: the grid size up to which the first of two launches handles a slice: sizes its shared memory;
// econ: the polynomials economised to degree 5, coefficients 6 and 7 zero -- the fused interpolation's tables)
cudaError_t launch_fft_filter(const float* grid, const float* D, int np, int ncap, const FPar* fp, const PolyWin& pw,
                              float* Q, int cap_hint, bool econ, const unsigned* flag16, cudaStream_t st);

// rows a5 + a7 by the NDFT on the kept band (ndft.cu; the paper's Gaussian engine): KW = padded band
// width (8, 16 or 32; ndft_width(K) = 0: too wide), what [np][2 KW] fp64 (zeroed by the caller)
constexpr int kNdftWidth = 32;
cudaError_t launch_ndft_spread(ZView zv, const float* w, int np, const FPar* fp, double* what, bool det,
                               const unsigned* flag16, cudaStream_t st);
constexpr int kNdftEvalGroup = 32;   // slices per k_ndft_eval CTA row (one TargetAcc group)
cudaError_t launch_ndft_eval(ZView zv, int np, const FPar* fp, const float* D, int dstride, const double* what,
                             TargetAcc acc, float* per_slice_out, bool accumulate_out, const unsigned* flag16,
                             cudaStream_t st);

// row a7 (+ Laplacian moment term) + slice accumulation:
//   per y_m: acc = sum_p [ Fourier interp + mom_coef * tau_p * S_moment ]
//   s64[m] += acc   (per_slice_out == nullptr)   or   per_slice_out[p*M + m] = t_{m,p}
struct EvalArgs {
  ZView zv;
  int np;
  const SliceTot* tot;   // slice totals (moment part)
  // Fourier part
  bool fourier;
  const FPar* fp;
  const float* Q;       // [np][q_stride(ncap)] per-cell interpolation polynomials (launch_fft_filter)
  int ncap;
  int w;                // window taps
  const unsigned* flag16;
  // Laplacian moment part: t += mom_coef * tau_p * sum_n w_n (z_n - z_m)^2
  bool moment;
  double mom_coef;
  // outputs
  TargetAcc acc;
  float* per_slice_out;
  bool accumulate_out;   // per_slice_out += t (after the sort path stored its part)
};
constexpr int kEvalGroup = 32;   // slices per eval CTA row in deterministic mode (one TargetAcc group)
cudaError_t launch_eval(const EvalArgs& a, bool det, cudaStream_t st);
cudaError_t launch_zero(void* p, size_t bytes, cudaStream_t st);
cudaError_t launch_finalize(const double* s64, int64_t M, double scale, float* s, cudaStream_t st);
// deterministic mode: s[m] = scale * sum_{g < G} part[g * M + m], the groups added in order
cudaError_t launch_finalize_det(const double* part, int G, int64_t M, double scale, float* s, cudaStream_t st);

}  // namespace sks
