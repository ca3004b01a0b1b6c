/*
 * sks.h -- sliced fast kernel summation on B200 (sm_100a), C ABI.
 *
 * Computes, for radial kernels K(x,y) = F(||x-y||), the kernel sums
 *     s_m = sum_{n=1}^{N} w_n F(||x_n - y_m||),  m = 1..M
 * by the paper's slicing method (Alg. 1):
 *     s_m ~= (1/P) sum_{p=1}^{P} t_{m,p},   t_{m,p} = sum_n w_n f(|<xi_p,x_n> - <xi_p,y_m>|)
 * with f the 1D counterpart of F (Table 1; App. C), xi_p iid uniform
 * directions on S^{d-1} drawn from `seed` (R1), and each 1D sum evaluated by
 *   - NEGDIST:   the exact sorting algorithm of Sec. 3.2 (Alg. 2), realised as a
 *                one-pass MSD (counting) sort + fp64 prefix sums;
 *   - GAUSSIAN / MATERN: fast Fourier summation on the torus (Sec. 3.1) with the
 *                NFFT (Remark P:519-525): spread -> FFT -> x D_k -> iFFT -> interpolate;
 *   - LAPLACIAN: the decomposition of Sec. 3.3: sorting part + Fourier part.
 *
 * Every compute step runs in this library's CUDA kernels (sm_100a).  There is no CPU fallback:
 * without a usable CUDA device every compute entry point returns SKS_ERR_CUDA.
 *
 * Conventions for all entry points
 *   - Point sets are row-major fp32: x is N x d (x[n*d + j]), y is M x d.  w is N fp32.
 *   - "DEVICE" pointers must be CUDA device (or managed) memory owned by the caller; the library
 *     never frees or retains them.  "HOST" pointers are ordinary host memory (pinned memory is
 *     faster for the _host variant).
 *   - The library allocates no memory on the hot path.  It keeps a small immutable per-process cache
 *     of device copies of the directions, keyed by (seed, P, d, p_begin, p_end), created on first use.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All work is enqueued on
 *     `stream` with no host synchronisation inside: the per-slice torus plan (row a2) is computed on the device
 *     from the projection epilogue's ranges, and the FP16x2 -> TF32x2 projection rerun is a device-predicated
 *     launch.  The device status of the call (non-finite projection, a plan beyond the built grid) sits in the
 *     first 48 bytes of the workspace.  By default the call ends with ONE synchronisation of `stream` that reads
 *     it back, so errors are returned by the call itself; with sks_options.async = 1 the call returns right after
 *     enqueueing and sks_sync_status(workspace, stream) reports the status later.
 *   - Return value: SKS_OK or an error status; sks_last_error() then returns a thread-local message.
 *     On error the contents of output buffers are unspecified.
 *   - Thread safety: calls on different threads may run concurrently (each thread uses its own helper streams
 *     and events; the direction / planner / graph caches are internally locked), also on different devices of
 *     one process.  Two calls must not share a workspace while either is in flight.
 */
#ifndef SKS_H_
#define SKS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SKS_OK = 0,
  SKS_ERR_INVALID = 1,      /* bad argument: sizes <= 0, NULL pointer, scale <= 0, bad slice range      */
  SKS_ERR_UNSUPPORTED = 2,  /* kernel kind not in sks_kind, Matern p outside [0, 8], or a plan that
                               exceeds the built limits (grid n > 16384)                                 */
  SKS_ERR_CUDA = 3,         /* CUDA runtime error (incl. no device / missing sm_100a support)            */
  SKS_ERR_WORKSPACE = 4,    /* workspace NULL or smaller than sks_workspace_size()                       */
  SKS_ERR_NONFINITE = 5     /* a projection was NaN/Inf (device flag, read at the call's synchronisation)  */
} sks_status;

typedef enum {
  SKS_GAUSSIAN = 0,   /* F(r) = exp(-r^2/(2 scale^2))                  Table 1                */
  SKS_NEGDIST = 1,    /* F(r) = -r                      (scale unused) Table 1                */
  SKS_LAPLACIAN = 2,  /* F(r) = exp(-r/scale): scale is a LENGTH, the paper's rate alpha = 1/scale
                         (R8)                                                    */
  SKS_MATERN = 3      /* Matern nu = matern_p + 1/2, length beta = scale (closed form P:1163)  */
} sks_kind;

typedef struct {
  int32_t kind;       /* sks_kind                                                   */
  int32_t matern_p;   /* SKS_MATERN only: nu = matern_p + 1/2, 0 <= matern_p <= 8   */
  double scale;       /* sigma | unused | ell | beta  (must be > 0 unless NEGDIST)  */
} sks_kernel;

/* Point sharding across GPUs (one process per GPU) for the large-N Fourier path.  The 1D fast Fourier summation
 * is linear in the sources up to the grids of Fourier data and pointwise in the targets after them, so
 * ranks may split the POINTS instead of the slices: every rank calls sks_sum with its own rows of x, w and y and the
 * full slice range, and the call invokes `exchange` (on the host, in enqueue order, for work on `stream`) where the
 * ranks' data must meet:
 *   SKS_XCHG_BCAST_F64  count doubles at dev_ptr: overwrite with rank 0's (the common centre mu of the range bound)
 *   SKS_XCHG_MAX_I32    count int32 at dev_ptr: element-wise maximum over the ranks (the 8 norm words; bit patterns
 *                       of non-negative floats, which order as integers)
 *   SKS_XCHG_SUM_F32    count floats at dev_ptr: element-wise sum over the ranks (a slice batch's NFFT grids)
 * dev_ptr points into the call's workspace.  The callback enqueues the collective after the work already enqueued on
 * `stream` (e.g. ncclAllReduce on that stream, or torch.distributed on the current stream) and returns 0, non-zero
 * on failure (the call then returns SKS_ERR_CUDA).  s receives the sums of the rank's own targets, equal to the
 * unsharded call's up to fp32 summation order of the grids.  Only the fused large-N path takes part (otherwise
 * SKS_ERR_UNSUPPORTED); not combinable with `graph` or `deterministic`. */
typedef enum { SKS_XCHG_BCAST_F64 = 0, SKS_XCHG_MAX_I32 = 1, SKS_XCHG_SUM_F32 = 2 } sks_exchange_op;
typedef int (*sks_exchange_fn)(void* user, int32_t op, void* dev_ptr, size_t count, void* stream);

/* Optional tuning knobs.  Pass NULL for the defaults (given in brackets). */
typedef struct {
  double eps;            /* [1e-6] absolute tail mass (f(0)-relative) of dropped Fourier coefficients and aliasing level
                            of the torus scaling (readings R3/R5 of P:339-349)             */
  int32_t window_w;      /* [6]  NFFT window width in grid cells (taps per point), 2..12 (the fused large-N path:
                            4..8, 10, 12; others take the stored-projection path).  6 is the narrowest width whose
                            worst-case aliasing bound meets the Fourier paths' 1e-4 tolerance with margin; measured
                            errors and times per width: DESIGN.md Sec. 7                                          */
  int32_t oversample;    /* [2]  NFFT oversampling factor n >= oversample * 2 * (k_max + 1)           */
  int32_t slice_batch;   /* [0 = auto] slices processed per batch (memory bound, Remark P:973-979)   */
  int32_t engine;        /* [0 = auto] Fourier engine for the Gaussian / Matern: 1 = NFFT (Remark P:519-525),
                            2 = NDFT on the kept band (the paper's Gaussian engine; at most 32
                            coefficients, else SKS_ERR_UNSUPPORTED); auto = NFFT (measured faster on B200)  */
  int32_t projection;    /* [0 = auto] row a1 arithmetic (R2), all fp32-accurate: 1 = BF16x3, 2 = TF32x2,
                            3 = FP16x2 (falls back to TF32x2 where it cannot run); auto picks by d and alignment.
                            The fused large-N path (Fourier kernels, N >= 2^18, d <= 128, d % 4 == 0, 16-byte
                            aligned rows) runs with auto or FP16x2 and computes FP16x2 with one power-of-two scale
                            per 8 points; 1 / 2 force the unfused path                                             */
  int32_t async;         /* [0] 1: return right after enqueueing (no synchronisation); the device status is read by
                            sks_sync_status(workspace, stream)                                                     */
  int32_t deterministic; /* [0] 1: bitwise run-to-run deterministic results: no floating-point atomics --
                            per-target sums of every slice group go to a partial-sum buffer added in a fixed order,
                            grids are accumulated by one CTA per slice, each sort bucket is taken in value order; the
                            fused large-N path is not used.  Same tolerances; slower where the atomics were spread  */
  int32_t graph;         /* [0] 1: replay the call as a CUDA graph (implies async).  The first call with a given set
                            of arguments (pointers, sizes, kernel, P, seed, range, options, stream) runs eagerly and
                            captures its launches; later identical calls launch the instantiated graph (one
                            cudaGraphLaunch): for launch-latency-bound problems (hard part 9)        */
  sks_exchange_fn exchange; /* [NULL] point sharding: the collective callback described above                      */
  void* exchange_user;      /* passed back to `exchange`                                                            */
} sks_options;

/* Diagnostic description of the last plan built on this thread (for reports and tests). */
typedef struct {
  int32_t path;          /* 0 = Fourier only, 1 = sort only, 2 = sort + Fourier                        */
  int32_t n_grid;        /* largest per-slice NFFT grid length n_p (power of two), 0 if no Fourier part */
  int32_t k_max;         /* largest |k| kept over the slices                                            */
  int32_t band_lo_min;   /* smallest lower band edge over the slices (Gaussian bands exclude 0..lo-1)   */
  int32_t window_w;      /* taps per point                                                              */
  int32_t spread_cells;  /* widest per-slice footprint W of the x points (cells)                        */
  int32_t n_buckets;     /* buckets of the counting sort (sort part), 0 if none                         */
  int32_t slice_batch;   /* slices per batch                                                            */
  int32_t n_batches;     /* batches in the call                                                         */
  int32_t launches;      /* CUDA kernels launched by the call                                           */
  double tau_min, tau_max;   /* torus scaling range over slices                                         */
  int32_t engine;        /* Fourier engine used: 0 none, 1 NFFT, 2 NDFT                                  */
  int32_t band_width;    /* widest kept band k_hi - k_lo + 1 over the slices                             */
  int32_t proj_mode;     /* projection arithmetic: 0 none (given projections), 2 BF16x3 (three bf16
                            MMAs per product), 3 TF32x2 (two tf32 MMAs per product), 4 FP16x2 (two fp16 MMAs per
                            product on 2^e-scaled points); reading R2                                             */
  int32_t fused;         /* 1: the sources' projections were spread and the targets' interpolated straight from the
                            tensor-core accumulators (rows a1 + a5 and a1 + a7 fused, never stored; SURVEY Sec. 8(f)
                            f2; proj_mode 4), 0: projections stored and re-read                                    */
} sks_plan_info;

/* Bytes of DEVICE workspace sks_sum needs for this problem (slice range [p_begin, p_end) of P).
 * Returns SKS_OK and writes *bytes, or an error for invalid arguments. */
sks_status sks_workspace_size(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t P,
                              int32_t p_begin, int32_t p_end, const sks_options* opt, size_t* bytes);

/* The hot path (Alg. 1) over slices p in [p_begin, p_end) of a P-direction estimate.
 *   x: DEVICE N x d fp32;  y: DEVICE M x d fp32;  w: DEVICE N fp32;
 *   s: DEVICE M fp32 out:  s_m = (1/P) sum_{p in [p_begin,p_end)} t_{m,p}.
 * With p_begin = 0, p_end = P this is the full estimate; partial ranges on several GPUs add up
 * (one all-reduce SUM of s) to the same estimate, because direction p depends only on (seed, p).
 * workspace: DEVICE, >= sks_workspace_size() bytes, 256-byte aligned. */
sks_status sks_sum(const float* x, int64_t N, const float* y, int64_t M, int32_t d, const float* w,
                   sks_kernel kernel, int32_t P, uint64_t seed, int32_t p_begin, int32_t p_end, float* s,
                   void* workspace, size_t workspace_bytes, const sks_options* opt, void* stream);

/* Same computation from HOST buffers x, y, w (copied in) to HOST s (copied out); blocks until s is
 * written.  workspace: DEVICE, >= sks_workspace_size_host() bytes. */
sks_status sks_workspace_size_host(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t P,
                                   int32_t p_begin, int32_t p_end, const sks_options* opt, size_t* bytes);
sks_status sks_sum_host(const float* x, int64_t N, const float* y, int64_t M, int32_t d, const float* w,
                        sks_kernel kernel, int32_t P, uint64_t seed, int32_t p_begin, int32_t p_end, float* s,
                        void* workspace, size_t workspace_bytes, const sks_options* opt, void* stream);

/* Directions of DESIGN.md R1 (host only, no GPU needed): for p in [p_begin, p_end),
 *   g_out[(p-p_begin)*d + j] = g_p[j]  (HOST, unnormalised N(0,1) draw rounded to bf16, exact in fp32)
 *   inv_norm_out[p-p_begin]   = 1/||g_p|| in fp64 (HOST);  xi_p = g_p * inv_norm_p. */
sks_status sks_directions(int32_t P, int32_t d, uint64_t seed, int32_t p_begin, int32_t p_end, float* g_out,
                          double* inv_norm_out);

/* Row a1 alone: z[(p-p_begin)*n + i] = <xi_p, pts_i>, pts DEVICE n x d fp32, z DEVICE fp32.
 * opt: NULL or options (only `projection` is used). */
sks_status sks_project(const float* pts, int64_t n, int32_t d, int32_t P, uint64_t seed, int32_t p_begin,
                       int32_t p_end, float* z, const sks_options* opt, void* stream);

/* Rows a2-a7 alone: per-slice 1D sums t[q*M + m] = sum_n w_n f(|zx[q*N+n] - zy[q*M+m]|) for q < n_slices
 * on given DEVICE projections zx (n_slices x N), zy (n_slices x M), DEVICE w (N); t DEVICE fp32 out.
 * f is the 1D counterpart of `kernel` in dimension d.  workspace: >= sks_workspace_size_1d(). */
sks_status sks_workspace_size_1d(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t n_slices,
                                 const sks_options* opt, size_t* bytes);
sks_status sks_sum_1d(const float* zx, const float* zy, const float* w, int64_t N, int64_t M, int32_t n_slices,
                      int32_t d, sks_kernel kernel, float* t, void* workspace, size_t workspace_bytes,
                      const sks_options* opt, void* stream);

/* Torus Fourier coefficients used by the planner (host only): out[k-k0] = c_k for k in [k0, k1] of the
 * periodised 1D counterpart on the torus of period 1/tau (Lemma 2.5 P:304-338 for GAUSSIAN; DESIGN.md
 * R7 / R7b closed forms for LAPLACIAN (smooth part of the Sec. 3.3 decomposition) and MATERN). */
sks_status sks_fourier_coeffs(sks_kernel kernel, int32_t d, double tau, int32_t k0, int32_t k1, double* out);

/* Plan of the last sks_sum / sks_sum_1d call on this thread.  The device-planned fields (n_grid, k_max,
 * band_lo_min, spread_cells, band_width, tau_min/max) are filled when the call's status was read back (the
 * default synchronous call, or sks_sync_status after an async one). */
sks_status sks_last_plan(sks_plan_info* info);

/* Synchronise `stream` and return the device status of the last call that used `workspace` (DEVICE pointer
 * passed to sks_sum / sks_sum_1d): SKS_OK, SKS_ERR_NONFINITE or SKS_ERR_UNSUPPORTED (a plan needing a grid
 * beyond the built limit, or an NDFT band wider than 32).  Also completes sks_last_plan's device fields. */
sks_status sks_sync_status(void* workspace, void* stream);

/* Opt-in measurement support (bench.py): while enabled, every kernel launch of sks_sum / sks_sum_1d is
 * bracketed by CUDA events recorded on the launch stream (negligible overhead, no synchronisation). */
sks_status sks_profile_enable(int32_t enable);
/* Accumulated device time (ms) and launch count per kernel slot since the last read; waits for the
 * recorded events, then resets.  n_slots >= SKS_PROFILE_SLOTS; slot names: sks_profile_names(). */
#define SKS_PROFILE_SLOTS 16
sks_status sks_profile_read(double* ms, int64_t* launches, int32_t n_slots);
/* Comma-separated slot names: "project,minmax,sortsum,plan_D,spread,fft_filter,eval,aux". */
const char* sks_profile_names(void);

/* Frees the library's device caches: the cached directions of every (device, seed, P, d, slice range) seen so far
 * (P_local x d x 8 bytes each), the planner's window tables and the CUDA graphs of sks_options.graph.  The caches
 * otherwise live until the process exits (calls with new (seed, P, d, range) keys add entries; each entry's first
 * call uploads it synchronously).  Waits for all work on the devices that hold entries; must not run while other
 * sks calls are in flight on any thread (their cached pointers would be freed).  The next call rebuilds what it
 * needs.  Returns SKS_OK or SKS_ERR_CUDA. */
sks_status sks_release_caches(void);

/* Thread-local message for the last non-OK status ("" if none). */
const char* sks_last_error(void);

/* Library version string. */
const char* sks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SKS_H_ */
