// api.cpp -- the C ABI of libsks (include/sks.h): validation, workspace carving, direction cache,
// slice batching and the per-batch kernel sequence of Alg. 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sks.h"
#include "host.h"
#include "kernels.h"

namespace {

// ---- opt-in kernel timing (sks_profile_*): event pairs per slot, resolved on read
using namespace sks;   // ProfSlot
struct Prof {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  double ms[PS_N] = {};
  int64_t cnt[PS_N] = {};
} g_prof;

bool capturing(cudaStream_t st) {   // no timing events inside a CUDA-graph capture
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {   // brackets one launch with events on its stream when profiling is on
  int slot;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int s, cudaStream_t stream) : slot(s), st(stream) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (!g_prof.on || capturing(st)) return;
    a = prof_event();
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, st);
    g_prof.pending.emplace_back(slot, a, b);
  }
};
#define PROF(slot) ProfScope prof_scope_##__LINE__(slot, st)

}  // namespace

namespace sks {
ProfMark prof_begin(int slot, cudaStream_t st) {
  ProfMark m{slot, st, nullptr};
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (!g_prof.on || capturing(st)) return m;
  m.a = prof_event();
  cudaEventRecord(m.a, st);
  return m;
}
void prof_end(const ProfMark& m) {
  if (!m.a) return;
  std::lock_guard<std::mutex> lk(g_prof.mu);
  cudaEvent_t b = prof_event();
  cudaEventRecord(b, m.st);
  g_prof.pending.emplace_back(m.slot, m.a, b);
}
}  // namespace sks

namespace {

thread_local std::string g_err;
thread_local sks_plan_info g_plan{};

sks_status fail(sks_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define SKS_CUDA(call)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) return fail(SKS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Opts {
  double eps = 1e-6;
  int w = 6;
  int os = 2;
  int batch = 0;
  int engine = 0;   // Fourier engine: 0 auto (= NFFT), 1 NFFT, 2 NDFT
  int proj = 0;     // row a1 variant: 0 auto, 1 BF16x3, 2 TF32x2, 3 FP16x2
  int async = 0;    // 1: enqueue only (status through sks_sync_status)
  int graph = 0;    // 1: replay a captured CUDA graph of the call (implies async)
  int det = 0;      // 1: bitwise run-to-run deterministic (no float atomics; fixed-order reductions)
  sks_exchange_fn xchg = nullptr;   // point sharding: the ranks' collective callback (sks.h)
  void* xuser = nullptr;
};

sks_status resolve_opts(const sks_options* o, Opts* r) {
  Opts d;
  if (o) {
    if (o->eps > 0) d.eps = o->eps;
    if (o->window_w) d.w = o->window_w;
    if (o->oversample) d.os = o->oversample;
    d.batch = o->slice_batch;
    if (d.w < 2 || d.w > 12) return fail(SKS_ERR_INVALID, "window_w must be in [2, 12]");
    if (d.os < 2 || d.os > 16) return fail(SKS_ERR_INVALID, "oversample must be in [2, 16]");
    if (d.batch < 0) return fail(SKS_ERR_INVALID, "slice_batch must be >= 0");
    d.engine = o->engine;
    if (d.engine < 0 || d.engine > 2) return fail(SKS_ERR_INVALID, "engine must be 0 (auto), 1 (NFFT) or 2 (NDFT)");
    d.proj = o->projection;
    if (d.proj < 0 || d.proj > 3)
      return fail(SKS_ERR_INVALID, "projection must be 0 (auto), 1 (BF16x3), 2 (TF32x2) or 3 (FP16x2)");
    d.graph = o->graph ? 1 : 0;
    d.async = (o->async || d.graph) ? 1 : 0;
    d.det = o->deterministic ? 1 : 0;
    d.xchg = o->exchange;
    d.xuser = o->exchange_user;
    if (d.xchg && (d.graph || d.det))
      return fail(SKS_ERR_INVALID, "exchange (point sharding) cannot be combined with graph or deterministic");
  }
  *r = d;
  return SKS_OK;
}

sks_status check_kernel(const sks_kernel& k) {
  if (k.kind < 0 || k.kind > 3) return fail(SKS_ERR_UNSUPPORTED, "unsupported kernel kind " + std::to_string(k.kind));
  if (k.kind != SKS_NEGDIST && !(k.scale > 0.0 && std::isfinite(k.scale)))
    return fail(SKS_ERR_INVALID, "kernel scale must be finite and > 0");
  if (k.kind == SKS_MATERN && (k.matern_p < 0 || k.matern_p > 8))
    return fail(SKS_ERR_UNSUPPORTED, "Matern p must be in [0, 8]");
  return SKS_OK;
}

struct Path {
  bool sort, fourier, moment;
};
Path path_of(int kind) {
  return Path{kind == SKS_NEGDIST || kind == SKS_LAPLACIAN, kind != SKS_NEGDIST, kind == SKS_LAPLACIAN};
}

constexpr int kNcapLog = 14;
constexpr int kNcap = 1 << kNcapLog;   // largest NFFT grid the kernels are built for (n_cap)
constexpr size_t kAlign = 256;
inline size_t al(size_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

// the call's status area at the start of the workspace: flag16 [4] (kernels.h), plan summary [8], + slack
constexpr size_t kStatusBytes = 64;

// workspace layout of one slice batch (offsets in bytes)
struct Layout {
  size_t status = 0, s64 = 0, mm = 0, Z = 0, xs3 = 0, part = 0, tot = 0, sp = 0, grid = 0, D = 0, fpar = 0, Q = 0,
         what = 0, bound = 0, wpad = 0, xh = 0, xl = 0, yh = 0, yl = 0, rsx = 0, rsy = 0, dpart = 0, total = 0;
  int dgroups = 0;   // deterministic mode: TargetAcc groups of the whole call
};

// deterministic mode: the TargetAcc groups (rows of the partial-sum buffer) a call writes -- the sort path's gather
// rows and the interpolation's slice groups, batch by batch
int det_groups(int64_t N, int64_t M, Path pt, int nslices, int batch) {
  int g = 0;
  for (int b0 = 0; b0 < nslices; b0 += batch) {
    const int nbat = std::min(batch, nslices - b0);
    if (pt.sort) g += sks::sortpart_acc_groups(N, M, nbat);
    if (pt.fourier || pt.moment) g += (nbat + sks::kEvalGroup - 1) / sks::kEvalGroup;
  }
  return g;
}

// The Laplacian's Fourier part (plan, spread, FFT: rows a2, a5, a6) does not read the sort stage's results (rows a3,
// a4), so it runs beside it on a side stream (forked after the projection, joined before the interpolation, which
// needs the sort stage's slice totals for the moment term).  One stream and two events per (thread, device), as the
// sort stage's helper streams (sortpart.cu): concurrent calls on different threads never share them.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false;
};
SideStream* side_stream(int dev) {
  thread_local std::map<int, SideStream> pools;
  SideStream& p = pools[dev];
  if (!p.ok)
    p.ok = cudaStreamCreateWithFlags(&p.s, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p.join, cudaEventDisableTiming) == cudaSuccess;
  return p.ok ? &p : nullptr;
}

// rows a1 + a5 and a1 + a7 fused (fused.cu) for the Fourier-only kernels when the points are many: the sources'
// projections are spread and the targets' interpolated straight from the tensor-core accumulators; no projection
// is stored.  The decision depends on the problem's shape only (never on data), so the workspace size is known up
// front (the run-time conditions -- TMA-readable points -- fall back to the stored-projection path, whose
// workspace the layout then also holds).
constexpr int64_t kFusedMinN = 1 << 18;
bool fused_shape(int64_t N, int d, Path pt, bool with_Z, int w) {
  return with_Z && pt.fourier && !pt.sort && N >= kFusedMinN && d <= 128 && d % 4 == 0 && w >= 4 && w != 9 && w != 11;
}

// fp32 -> IEEE binary16, round to nearest even (host; |v| < 65504 here)
uint16_t to_half_rne(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  const uint32_t sign = (u >> 16) & 0x8000u;
  const float a = std::fabs(v);
  if (a >= 65520.0f) return static_cast<uint16_t>(sign | 0x7c00u);
  if (a < 6.103515625e-05f) {   // subnormal: multiple of 2^-24, rounded to nearest even
    const float q = a * 16777216.0f;
    return static_cast<uint16_t>(sign | static_cast<uint32_t>(std::nearbyint(q)));
  }
  uint32_t au;
  std::memcpy(&au, &a, 4);
  const uint32_t r = au + 0xfffu + ((au >> 13) & 1u);   // round the low 13 mantissa bits to nearest even
  const uint32_t e = (r >> 23) - 127 + 15, m = (r >> 13) & 0x3ffu;
  return static_cast<uint16_t>(sign | (e << 10) | m);
}

// row a1 variant (reading R2).  TF32x2 reads the fp32 points once (TMA: the raw tile is the hi operand) and
// needs no split buffer; FP16x2 has the same precision at twice the MMA rate but a sampled point scale, so it is
// taken where the GEMM is compute-bound (d >= 256).  Points TMA cannot read (unaligned, d % 4 != 0): TF32x2 with
// the converters loading the points below d = 256, BF16x3 (split pass + three bf16 MMAs) above (measured cfg3
// 0.56 vs 0.59 ms, cfg4 1.64 vs 1.79 ms for TF32x2 vs BF16x3 with TMA; without TMA BF16x3 wins above d = 256).
// sks_options.projection forces a variant (tests of every variant).
enum ProjMode { PM_AUTO = 0, PM_BF16X3 = 1, PM_TF32X2 = 2, PM_FP16X2 = 3 };

// the variant that sizes the workspace (BF16x3 needs the split buffer)
ProjMode proj_mode(int d, int forced) {
  if (forced) return static_cast<ProjMode>(forced);
  return d <= 256 ? PM_TF32X2 : PM_BF16X3;
}

ProjMode proj_mode_call(int d, int forced, const float* x, int64_t N, const float* y, int64_t M) {
  const bool tma = sks::proj_tf32_tma_ok(x, N, y, M, d);
  if (forced) {
    ProjMode pm = static_cast<ProjMode>(forced);
    if (pm == PM_FP16X2 && !tma) pm = PM_TF32X2;
    return pm;
  }
  if (tma) return d >= 256 ? PM_FP16X2 : PM_TF32X2;
  return proj_mode(d, 0);
}

// leading dimension of the slice-major projections Z: a multiple of 4 floats (16-byte rows for TMA stores)
inline int64_t zld(int64_t N, int64_t M) { return (N + M + 3) / 4 * 4; }

Layout make_layout(int64_t N, int64_t M, Path pt, int nbat, bool with_Z, int d, int proj, bool fused, int dgroups = 0) {
  Layout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += al(bytes);
    return at;
  };
  L.status = take(kStatusBytes);
  L.s64 = take(sizeof(double) * M);
  L.mm = take(sizeof(unsigned) * 4 * nbat);
  if (with_Z) {
    L.Z = take(sizeof(float) * zld(N, M) * nbat);   // (fused calls do not touch it unless they fall back)
    if (proj_mode(d, proj) == PM_BF16X3) {
      L.xs3 = take(sizeof(uint16_t) * 3 * static_cast<size_t>(sks::proj_tc_dpad(d)) * (N + M));
      L.part = take(sks::proj_tc_part_bytes(nbat));
    }
  }
  if (pt.sort || pt.moment) {
    L.tot = take(sizeof(sks::SliceTot) * static_cast<size_t>(nbat));
    L.sp = take(sks::sortpart_bytes(N, M, nbat));
  }
  if (pt.fourier) {
    L.grid = take(sizeof(float) * kNcap * static_cast<size_t>(nbat));
    L.D = take(sizeof(float) * (kNcap / 2 + 1) * static_cast<size_t>(nbat));
    L.fpar = take(sizeof(sks::FPar) * nbat);
    L.Q = take(sizeof(float) * sks::q_stride(kNcap) * static_cast<size_t>(nbat));
    L.what = take(sizeof(double) * 2 * sks::kNdftWidth * static_cast<size_t>(nbat));
    if (fused) {
      L.bound = take(sks::source_bound_bytes(d));
      // both point sets as FP16x2 operands (hi, lo: fp16 [rows][dp16]) and their per-8-row scales (source prep)
      const size_t dp16 = static_cast<size_t>(sks::fused_dp16(d));
      L.xh = take(sizeof(uint16_t) * static_cast<size_t>(N) * dp16);
      L.xl = take(sizeof(uint16_t) * static_cast<size_t>(N) * dp16);
      L.yh = take(sizeof(uint16_t) * static_cast<size_t>(M) * dp16);
      L.yl = take(sizeof(uint16_t) * static_cast<size_t>(M) * dp16);
      L.rsx = take(sizeof(float) * static_cast<size_t>((N + 127) / 128 * 16));   // per 8-row group (whole tiles)
      L.wpad = take(sizeof(float) * static_cast<size_t>((N + 127) / 128 * 128));
      L.rsy = take(sizeof(float) * static_cast<size_t>((M + 127) / 128 * 16));
    }
  }
  if (dgroups) {
    L.dpart = take(sizeof(double) * static_cast<size_t>(M) * dgroups);
    L.dgroups = dgroups;
  }
  L.total = o;
  return L;
}

int choose_batch(int64_t N, int64_t M, Path pt, int np, bool with_Z, int req, int d, int proj, bool fused) {
  if (req > 0) return std::min(req, np);
  // auto: all local slices unless the batch working set would exceed 64 GiB of HBM
  const size_t budget = size_t(64) << 30;
  int b = np;
  while (b > 1 && make_layout(N, M, pt, b, with_Z, d, proj, fused).total > budget) b = (b + 1) / 2;
  return b;
}

// ---- direction cache (device copies; immutable once created)
struct DirEntry {
  float* inv = nullptr;    // np
  void* g3 = nullptr;      // np x dp bf16: g zero padded (BF16x3 tensor-core operand)
  int K3 = 0;              // dp
  float* g32 = nullptr;    // np x dp32 fp32: g zero padded to 32 (TF32x2 operand; bf16-exact, so tf32-exact)
  void* g16 = nullptr;     // np x K3 fp16: 2^8 g (FP16x2 operand; exact but for |g| < 2^-22)
  int K32 = 0;             // dp32
};
std::mutex g_dir_mu;
std::map<std::tuple<int, uint64_t, int, int, int, int>, DirEntry> g_dirs;

sks_status get_dirs(int P, int d, uint64_t seed, int p0, int p1, DirEntry* out) {
  int dev = 0;
  SKS_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, seed, P, d, p0, p1);
  std::lock_guard<std::mutex> lk(g_dir_mu);
  auto it = g_dirs.find(key);
  if (it != g_dirs.end()) {
    *out = it->second;
    return SKS_OK;
  }
  const int np = p1 - p0;
  std::vector<float> g(static_cast<size_t>(np) * d);
  std::vector<double> inv(np);
  sks::make_directions(P, d, seed, p0, p1, g.data(), inv.data());
  std::vector<float> invf(np);
  for (int i = 0; i < np; ++i) invf[i] = static_cast<float>(inv[i]);
  DirEntry e;
  SKS_CUDA(cudaMalloc(&e.inv, sizeof(float) * np));
  SKS_CUDA(cudaMemcpy(e.inv, invf.data(), sizeof(float) * np, cudaMemcpyHostToDevice));
  const int dp = sks::proj_tc_dpad(d);
  e.K3 = dp;
  std::vector<uint16_t> g3(static_cast<size_t>(np) * e.K3, 0);
  for (int p = 0; p < np; ++p)
    for (int j = 0; j < d; ++j) {
      uint32_t u;
      std::memcpy(&u, &g[static_cast<size_t>(p) * d + j], 4);
      g3[static_cast<size_t>(p) * e.K3 + j] = static_cast<uint16_t>(u >> 16);   // exact: g is bf16 (R1)
    }
  SKS_CUDA(cudaMalloc(&e.g3, sizeof(uint16_t) * g3.size()));
  SKS_CUDA(cudaMemcpy(e.g3, g3.data(), sizeof(uint16_t) * g3.size(), cudaMemcpyHostToDevice));
  e.K32 = sks::proj_tf32_dpad(d);
  std::vector<float> g32(static_cast<size_t>(np) * e.K32, 0.f);
  for (int p = 0; p < np; ++p)
    for (int j = 0; j < d; ++j) g32[static_cast<size_t>(p) * e.K32 + j] = g[static_cast<size_t>(p) * d + j];
  SKS_CUDA(cudaMalloc(&e.g32, sizeof(float) * g32.size()));
  SKS_CUDA(cudaMemcpy(e.g32, g32.data(), sizeof(float) * g32.size(), cudaMemcpyHostToDevice));
  std::vector<uint16_t> g16(static_cast<size_t>(np) * e.K3, 0);
  for (int p = 0; p < np; ++p)
    for (int j = 0; j < d; ++j) g16[static_cast<size_t>(p) * e.K3 + j] = to_half_rne(256.0f * g[static_cast<size_t>(p) * d + j]);
  SKS_CUDA(cudaMalloc(&e.g16, sizeof(uint16_t) * g16.size()));
  SKS_CUDA(cudaMemcpy(e.g16, g16.data(), sizeof(uint16_t) * g16.size(), cudaMemcpyHostToDevice));
  g_dirs[key] = e;
  *out = e;
  return SKS_OK;
}

// ---- planner constants: data-independent, cached per device (host fp64 + one upload of the window table)
struct PlanEntry {
  sks::PlanConst pc{};
  sks::PolyWin pw{};
  float* phi2inv = nullptr;   // device [kNcap / 2 + 1]
};
std::mutex g_plan_mu;
std::map<std::tuple<int, int, int, double, int, double, int, int>, PlanEntry> g_plans;

sks::CoeffConst coeff_const(const sks_kernel& k, int d) {
  sks::CoeffConst c{};
  c.kind = k.kind;
  c.d = d;
  c.scale = k.scale;
  const double PI = 3.14159265358979323846;
  if (k.kind == SKS_GAUSSIAN) c.logpref = std::log(d * PI / std::sqrt(2.0)) - std::lgamma(0.5 * d + 1.0);
  if (k.kind == SKS_LAPLACIAN) {
    c.logpref = std::log(2.0 * sks::cd(d));
    c.lap_A = sks::cd(d) / k.scale;
  }
  if (k.kind == SKS_MATERN) {
    const double nu = k.matern_p + 0.5;
    c.nu = nu;
    c.logpref = 0.5 * d * std::log(PI) - std::lgamma(0.5 * d) + d * std::log(2.0) + 0.5 * d * std::log(PI) +
                std::lgamma(nu + 0.5 * d) + nu * std::log(2.0 * nu) - std::lgamma(nu);
  }
  return c;
}

sks::PolyWin poly_win(const sks::WindowTables& wt) {
  sks::PolyWin pw{};
  pw.w = wt.w;
  for (size_t i = 0; i < sizeof(pw.c) / sizeof(float); ++i) pw.c[i] = i < wt.poly.size() ? wt.poly[i] : 0.f;
  // centered even / odd form of taps j < w/2 (fp64 binomial re-expansion of the power basis about f = 1/2)
  constexpr int D = sks::PW_D;
  static_assert(D == 7, "even/odd split assumes degree 7");
  for (int j = 0; j < (wt.w + 1) / 2 && j < 6; ++j) {
    double dm[D + 1] = {0};
    for (int k = 0; k <= D; ++k) {
      const double ck = (static_cast<size_t>(j) * (D + 1) + k < wt.poly.size()) ? wt.poly[j * (D + 1) + k] : 0.0;
      double binom = 1.0;   // C(k, m) (1/2)^{k - m} u^m
      for (int m = 0; m <= k; ++m) {
        dm[m] += ck * binom * std::pow(0.5, k - m);
        binom = binom * (k - m) / (m + 1);
      }
    }
    for (int i = 0; i < 4; ++i) {
      pw.eo[j][i] = static_cast<float>(dm[2 * i]);
      pw.eo[j][4 + i] = static_cast<float>(dm[2 * i + 1]);
    }
  }
  return pw;
}

sks_status get_plan(const sks_kernel& k, int d, const Opts& o, bool ndft, PlanEntry* out) {
  int dev = 0;
  SKS_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, k.kind, k.kind == SKS_MATERN ? k.matern_p : 0, k.scale, d, o.eps, o.w, o.os);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    PlanEntry e;
    const sks::KernelModel km{k.kind, k.matern_p, k.scale, d};
    e.pc.cc = coeff_const(k, d);
    e.pc.reps = sks::decay_radius(km, o.eps);
    e.pc.eps = o.eps;
    e.pc.os = o.os;
    e.pc.w = o.w;
    e.pc.ncap_log = kNcapLog;
    const sks::WindowTables& wt = sks::window_tables(o.w, o.os, kNcap);
    if (!(wt.poly_err < 1e-4))
      return fail(SKS_ERR_UNSUPPORTED, "window polynomial fit failed (error " + std::to_string(wt.poly_err) + ")");
    e.pw = poly_win(wt);
    SKS_CUDA(cudaMalloc(&e.phi2inv, sizeof(float) * wt.phi2inv.size()));
    SKS_CUDA(cudaMemcpy(e.phi2inv, wt.phi2inv.data(), sizeof(float) * wt.phi2inv.size(), cudaMemcpyHostToDevice));
    it = g_plans.emplace(key, e).first;
  }
  *out = it->second;
  out->pc.ndft = ndft ? 1 : 0;
  return SKS_OK;
}

// ---- pinned host staging for the status readback (per thread)
struct Staging {
  void* p = nullptr;
  ~Staging() {
    if (p) cudaFreeHost(p);
  }
};
thread_local Staging g_stage;

sks_status validate_common(int64_t N, int64_t M, int32_t d, const sks_kernel& k, int32_t P, int32_t p0, int32_t p1) {
  if (N <= 0 || M <= 0 || d <= 0) return fail(SKS_ERR_INVALID, "N, M and d must be > 0");
  // the sort path and the per-target indices hold N and M in 32-bit integers
  if (N > INT32_MAX || M > INT32_MAX) return fail(SKS_ERR_INVALID, "N and M must be < 2^31");
  if (P <= 0 || p0 < 0 || p1 > P || p0 >= p1) return fail(SKS_ERR_INVALID, "slice range must satisfy 0 <= p_begin < p_end <= P");
  return check_kernel(k);
}

// the batched pipeline shared by sks_sum and sks_sum_1d: enqueues every kernel of the call on `st` with no host
// synchronisation (the device planner takes the projection ranges straight from the epilogue); the status words
// at the start of the workspace are read back by finish_call / sks_sync_status
struct Problem {
  int64_t N, M;
  int d;
  sks_kernel k;
  int nslices;
  bool with_Z;
};

sks_status enqueue_call(const Problem& pr, const Opts& o, const float* x, const float* y, const float* w,
                        const DirEntry* dirs, const float* zx_in, const float* zy_in, float* s_out, float* t_out,
                        double inv_P, void* workspace, size_t ws_bytes, cudaStream_t st, sks_plan_info* info_out) {
  const Path pt = path_of(pr.k.kind);
  const bool fshape = fused_shape(pr.N, pr.d, pt, pr.with_Z, o.w) && o.engine != 2 && !o.det;
  const int batch = choose_batch(pr.N, pr.M, pt, pr.nslices, pr.with_Z, o.batch, pr.d, o.proj, fshape);
  const bool det = o.det && s_out;   // (per-slice outputs of sks_sum_1d have no cross-slice sums)
  const Layout L = make_layout(pr.N, pr.M, pt, batch, pr.with_Z, pr.d, o.proj, fshape,
                               det ? det_groups(pr.N, pr.M, pt, pr.nslices, batch) : 0);
  if (!workspace || ws_bytes < L.total)
    return fail(SKS_ERR_WORKSPACE, "workspace too small: need " + std::to_string(L.total) + " bytes");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return fail(SKS_ERR_INVALID, "workspace must be 256-byte aligned");
  char* ws = static_cast<char*>(workspace);
  const double cdd = sks::cd(pr.d);
  const bool ndft = pt.fourier && o.engine == 2 && (pr.k.kind == SKS_GAUSSIAN || pr.k.kind == SKS_MATERN);
  if (o.engine == 2 && !ndft)
    return fail(SKS_ERR_UNSUPPORTED, "NDFT engine: Gaussian / Matern with at most 32 kept coefficients only");
  PlanEntry plan;
  if (pt.fourier) {
    sks_status s = get_plan(pr.k, pr.d, o, ndft, &plan);
    if (s != SKS_OK) return s;
  }
  unsigned* flag16 = reinterpret_cast<unsigned*>(ws + L.status);
  unsigned* summary = flag16 + 4;
  int launches = 0, nbatches = 0, dgoff = 0;
  {   // flag words, fp64 target sums and the first batch's ranges in one launch
    ProfScope ps(PS_AUX, st);
    SKS_CUDA(sks::launch_prologue(flag16, s_out ? reinterpret_cast<double*>(ws + L.s64) : nullptr, pr.M,
                                  reinterpret_cast<unsigned*>(ws + L.mm), std::min(batch, pr.nslices), st));
  }
  launches += 1;
  const ProjMode pm = pr.with_Z ? proj_mode_call(pr.d, o.proj, x, pr.N, y, pr.M) : PM_AUTO;
  // fused path: the shape qualifies, the points are 16-byte aligned rows, and the projection variant is the automatic
  // choice or FP16x2 (the fused kernels compute FP16x2 with per-tile scales; d <= 128)
  const bool fused = fshape && (o.proj == 0 || o.proj == PM_FP16X2) && s_out && sks::fused_spread_ok(pr.d, x) &&
                     sks::fused_spread_ok(pr.d, y);
  if (o.xchg && !fused)
    return fail(SKS_ERR_UNSUPPORTED,
                "exchange (point sharding): the fused large-N Fourier path only (Gaussian / Matern, local N >= 2^18, "
                "d <= 128, d % 4 == 0, 16-byte aligned rows)");
  auto exchange = [&](int op, void* ptr, size_t count, cudaStream_t s) -> sks_status {
    if (o.xchg && o.xchg(o.xuser, op, ptr, count, s) != 0) return fail(SKS_ERR_CUDA, "exchange callback failed");
    return SKS_OK;
  };
  const bool tc = pr.with_Z && pm == PM_BF16X3;
  const bool tf = pr.with_Z && pm == PM_TF32X2;
  const bool th = pr.with_Z && pm == PM_FP16X2;
  if (tc) {
    ProfScope ps(PS_SPLIT, st);
    SKS_CUDA(sks::launch_split3(x, pr.N, y, pr.M, pr.d, ws + L.xs3, st));
    ++launches;
  }
  if (fused) {   // direction-independent: the sources' centre and radius, the targets' radius, FP16x2 operands
    ProfScope ps(PS_MINMAX, st);
    double* mu = reinterpret_cast<double*>(ws + L.bound);
    unsigned* nb = reinterpret_cast<unsigned*>(ws + L.bound + sks::source_bound_bytes(pr.d) - 32);
    // (point sharding: every rank bounds its points about rank 0's centre, the bounds' maxima cover all points)
    SKS_CUDA(sks::launch_source_mean(x, pr.N, pr.d, mu, nb, st));
    if (exchange(SKS_XCHG_BCAST_F64, mu, static_cast<size_t>(pr.d), st) != SKS_OK) return SKS_ERR_CUDA;
    SKS_CUDA(sks::launch_source_prep(x, pr.N, y, pr.M, pr.d, mu, nb, reinterpret_cast<uint16_t*>(ws + L.xh),
                                     reinterpret_cast<uint16_t*>(ws + L.xl), reinterpret_cast<float*>(ws + L.rsx),
                                     reinterpret_cast<uint16_t*>(ws + L.yh), reinterpret_cast<uint16_t*>(ws + L.yl),
                                     reinterpret_cast<float*>(ws + L.rsy), w, reinterpret_cast<float*>(ws + L.wpad), st));
    if (exchange(SKS_XCHG_MAX_I32, nb, 8, st) != SKS_OK) return SKS_ERR_CUDA;
    launches += 4;
  }
  for (int b0 = 0; b0 < pr.nslices; b0 += batch) {
    const int nbat = std::min(batch, pr.nslices - b0);
    ++nbatches;
    unsigned* mm = reinterpret_cast<unsigned*>(ws + L.mm);
    int* flag = reinterpret_cast<int*>(flag16);
    if (b0 > 0) {   // (the first batch's ranges are initialised by the prologue)
      ProfScope ps(PS_AUX, st);
      SKS_CUDA(sks::launch_init_minmax(mm, nbat, st));
      ++launches;
    }
    sks::ZView zv;
    if (fused) {   // nothing stored: both point sets are projected inside the fused kernels below
      zv = sks::ZView{nullptr, nullptr, 0, 0, pr.N, pr.M};
    } else if (pr.with_Z) {
      float* Z = reinterpret_cast<float*>(ws + L.Z);
      const int64_t ldz = zld(pr.N, pr.M);
      ProfScope ps(PS_PROJECT, st);
      const int chunks = (nbat + 1023) / 1024;
      if (tc) {
        SKS_CUDA(sks::launch_project_tc(ws + L.xs3, pr.N + pr.M, pr.N, pr.d,
                                        static_cast<const uint16_t*>(dirs->g3) + static_cast<int64_t>(b0) * dirs->K3,
                                        nbat, dirs->inv + b0, Z, ldz, mm, flag, ws + L.part, st));
        launches += chunks;
      } else if (tf) {
        SKS_CUDA(sks::launch_project_tf32(x, pr.N, y, pr.M, pr.d, dirs->g32 + static_cast<int64_t>(b0) * dirs->K32,
                                          nbat, dirs->inv + b0, Z, ldz, mm, flag, nullptr, st));
        launches += chunks;
      } else {   // FP16x2, then -- only if a point fell outside the fp16 range (flag) -- the same batch on TF32x2
        SKS_CUDA(sks::launch_project_f16(x, pr.N, y, pr.M, pr.d,
                                         static_cast<const uint16_t*>(dirs->g16) + static_cast<int64_t>(b0) * dirs->K3,
                                         nbat, dirs->inv + b0, Z, ldz, mm, flag, flag16 + 1, st));
        SKS_CUDA(sks::launch_rerun_prep(flag16, mm, nbat, st));
        SKS_CUDA(sks::launch_project_tf32(x, pr.N, y, pr.M, pr.d, dirs->g32 + static_cast<int64_t>(b0) * dirs->K32,
                                          nbat, dirs->inv + b0, Z, ldz, mm, flag, flag16 + 3, st));
        launches += 2 + 2 * chunks;
      }
      zv = sks::ZView{Z, Z + pr.N, ldz, ldz, pr.N, pr.M};
    } else {
      zv = sks::ZView{zx_in + static_cast<int64_t>(b0) * pr.N, zy_in + static_cast<int64_t>(b0) * pr.M, pr.N, pr.M,
                      pr.N, pr.M};
      ProfScope ps(PS_MINMAX, st);
      SKS_CUDA(sks::launch_minmax(zv, nbat, mm, flag, st));
      ++launches;
    }
    double* s64 = s_out ? reinterpret_cast<double*>(ws + L.s64) : nullptr;
    float* tps = t_out ? t_out + static_cast<int64_t>(b0) * pr.M : nullptr;
    // where the per-target sums go: fp64 atomics into s64, or (deterministic mode) the next rows of the partial-sum
    // buffer, added in order by the finalize kernel
    auto target_acc = [&](int groups) {
      sks::TargetAcc ta{s64, nullptr, pr.M, 0};
      if (det) {
        ta.part = reinterpret_cast<double*>(ws + L.dpart);
        ta.goff = dgoff;
        dgoff += groups;
      }
      return ta;
    };
    sks::EvalArgs ea{};
    ea.zv = zv;
    ea.np = nbat;
    ea.flag16 = flag16;
    // the Laplacian's Fourier part beside the sort stage (SideStream above)
    cudaStream_t fst = st;
    SideStream* side = nullptr;
    if (pt.sort && pt.fourier && !ndft) {
      int dev = 0;
      SKS_CUDA(cudaGetDevice(&dev));
      side = side_stream(dev);
      if (side) {
        SKS_CUDA(cudaEventRecord(side->fork, st));
        SKS_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
        fst = side->s;
      }
    }
    if (pt.sort) {
      // negdist: f = -c_d r; Laplacian sort part K2 = -alpha ||.||  -> -alpha c_d r (R7)
      sks::SortPartArgs sa{};
      sa.zv = zv;
      sa.w = w;
      sa.np = nbat;
      sa.mm = mm;
      sa.tot = reinterpret_cast<sks::SliceTot*>(ws + L.tot);
      sa.coef = (pr.k.kind == SKS_NEGDIST) ? cdd : cdd / pr.k.scale;
      sa.acc = target_acc(sks::sortpart_acc_groups(pr.N, pr.M, nbat));
      sa.per_slice_out = tps;
      sa.det = det;
      {
        ProfScope ps(PS_SORT, st);   // the whole sort stage (fork .. join); its kernels also time themselves
        SKS_CUDA(sks::launch_sortpart(sa, ws + L.sp, st));
      }
      launches += sks::sortpart_launches_per_group(pr.N, pr.M) * sks::sortpart_groups(pr.N, pr.M, nbat);
      ea.tot = sa.tot;
    }
    if (pt.fourier) {
      sks::FPar* fp = reinterpret_cast<sks::FPar*>(ws + L.fpar);
      float* grid = reinterpret_cast<float*>(ws + L.grid);
      if (fused) {   // both point sets' range bounds in place of their exact ranges (fused.cu; the planner's input)
        ProfScope ps(PS_PLAN, fst);
        SKS_CUDA(sks::launch_bound_ranges(dirs->g32 + static_cast<int64_t>(b0) * dirs->K32, dirs->K32, pr.d,
                                          dirs->inv + b0, nbat, reinterpret_cast<const double*>(ws + L.bound),
                                          reinterpret_cast<const unsigned*>(ws + L.bound + sks::source_bound_bytes(pr.d) - 32),
                                          mm, flag16, fst));
        launches += 1;
      }
      {
        ProfScope ps(PS_PLAN, fst);
        SKS_CUDA(sks::launch_plan(mm, nbat, plan.pc, plan.phi2inv, fp, reinterpret_cast<float*>(ws + L.D), grid, flag16,
                                  summary, fst));
        launches += 1;
      }
      if (ndft) {
        double* what = reinterpret_cast<double*>(ws + L.what);
        {
          ProfScope ps(PS_AUX, fst);
          SKS_CUDA(sks::launch_zero(what, al(sizeof(double) * 2 * sks::kNdftWidth * static_cast<size_t>(nbat)), fst));
        }
        {
          ProfScope ps(PS_NDFT_SPREAD, fst);
          SKS_CUDA(sks::launch_ndft_spread(zv, w, nbat, fp, what, det, flag16, fst));
        }
        {
          ProfScope ps(PS_NDFT_EVAL, fst);
          SKS_CUDA(sks::launch_ndft_eval(zv, nbat, fp, reinterpret_cast<const float*>(ws + L.D), kNcap / 2 + 1, what,
                                         target_acc((nbat + sks::kNdftEvalGroup - 1) / sks::kNdftEvalGroup), tps,
                                         pt.sort, flag16, fst));
        }
        launches += nbat <= 148 ? 2 : 3;
        continue;
      }
      if (fused) {
        ProfScope ps(PS_SPREAD, fst);
        SKS_CUDA(sks::launch_proj_spread(reinterpret_cast<const uint16_t*>(ws + L.xh),
                                         reinterpret_cast<const uint16_t*>(ws + L.xl),
                                         reinterpret_cast<const float*>(ws + L.rsx), pr.N, pr.d,
                                         static_cast<const uint16_t*>(dirs->g16) + static_cast<int64_t>(b0) * dirs->K3,
                                         dirs->K3, dirs->inv + b0, nbat, reinterpret_cast<const float*>(ws + L.wpad), fp,
                                         plan.pw, kNcap, grid, flag16, fst));
        // (point sharding: the grids of all ranks' sources)
        if (exchange(SKS_XCHG_SUM_F32, grid, static_cast<size_t>(nbat) * kNcap, fst) != SKS_OK) return SKS_ERR_CUDA;
      } else {
        ProfScope ps(PS_SPREAD, fst);
        SKS_CUDA(sks::launch_spread(zv, w, nbat, fp, kNcap, plan.pw, pr.k.kind == SKS_LAPLACIAN, det, grid, flag16, fst));
      }
      {
        ProfScope ps(PS_FFT, fst);
        // the first tier's grid capacity: the Laplacian's smooth part needs wide bands (n_p ~ 2048-4096 on the
        // BJ / paper workloads), the Gaussian / Matern narrow ones (n_p ~ 64-1024)
        SKS_CUDA(sks::launch_fft_filter(grid, reinterpret_cast<const float*>(ws + L.D), nbat, kNcap, fp, plan.pw,
                                        reinterpret_cast<float*>(ws + L.Q), pr.k.kind == SKS_LAPLACIAN ? 4096 : 2048,
                                        fused, flag16, fst));
      }
      launches += (nbat <= 148 ? 2 : 3) + (fused ? 2 : 0);   // (fused spread: three variants, one per footprint class)
      if (side) {   // join: the interpolation (on st, after the sort stage) waits for the Fourier part
        SKS_CUDA(cudaEventRecord(side->join, fst));
        SKS_CUDA(cudaStreamWaitEvent(st, side->join, 0));
      }
      ea.fourier = true;
      ea.fp = fp;
      ea.Q = reinterpret_cast<const float*>(ws + L.Q);
      ea.ncap = kNcap;
      ea.w = o.w;
    }
    if (pt.moment) {
      ea.moment = true;
      ea.mom_coef = cdd / pr.k.scale;   // + alpha c_d tau sum_n w_n (z_n - z_m)^2   (R7)
    }
    ea.per_slice_out = tps;
    ea.accumulate_out = pt.sort;
    if (pt.fourier || pt.moment) ea.acc = fused ? sks::TargetAcc{s64, nullptr, pr.M, 0}
                                                : target_acc((nbat + sks::kEvalGroup - 1) / sks::kEvalGroup);
    if (fused) {
      ProfScope ps(PS_EVAL, st);
      SKS_CUDA(sks::launch_proj_eval(reinterpret_cast<const uint16_t*>(ws + L.yh),
                                     reinterpret_cast<const uint16_t*>(ws + L.yl),
                                     reinterpret_cast<const float*>(ws + L.rsy), pr.M, pr.d,
                                     static_cast<const uint16_t*>(dirs->g16) + static_cast<int64_t>(b0) * dirs->K3,
                                     dirs->K3, dirs->inv + b0, nbat, ea.fp, ea.Q, kNcap, o.w, s64, flag16, st));
      launches += 1;
    } else if (pt.fourier || pt.moment) {
      ProfScope ps(PS_EVAL, st);
      SKS_CUDA(sks::launch_eval(ea, det, st));
      ++launches;
    }
  }
  if (s_out) {
    ProfScope ps(PS_AUX, st);
    if (det)
      SKS_CUDA(sks::launch_finalize_det(reinterpret_cast<const double*>(ws + L.dpart), dgoff, pr.M, inv_P, s_out, st));
    else
      SKS_CUDA(sks::launch_finalize(reinterpret_cast<const double*>(ws + L.s64), pr.M, inv_P, s_out, st));
    ++launches;
  }
  sks_plan_info info{};
  info.path = pt.fourier ? (pt.sort ? 2 : 0) : 1;
  info.engine = pt.fourier ? (ndft ? 2 : 1) : 0;
  info.window_w = pt.fourier ? o.w : 0;
  info.n_buckets = (pt.sort || pt.moment) ? sks::sortpart_dims(pr.N, pr.M).NH : 0;
  info.slice_batch = batch;
  info.n_batches = nbatches;
  info.launches = launches;
  info.proj_mode = !pr.with_Z ? 0 : fused ? 4 : tc ? 2 : tf ? 3 : 4;
  info.fused = fused ? 1 : 0;
  *info_out = info;
  return SKS_OK;
}

// read the call's status words (one 48-byte readback and a stream synchronisation) into a status and the plan
// summary; `info` holds the host-side fields of the call
sks_status read_status(const void* workspace, cudaStream_t st, sks_plan_info* info) {
  if (!g_stage.p) SKS_CUDA(cudaHostAlloc(&g_stage.p, kStatusBytes, cudaHostAllocDefault));
  unsigned* h = static_cast<unsigned*>(g_stage.p);
  SKS_CUDA(cudaMemcpyAsync(h, workspace, 48, cudaMemcpyDeviceToHost, st));
  SKS_CUDA(cudaStreamSynchronize(st));
  if (info && info->path != 1) {   // Fourier plan summary (plan.cu)
    const unsigned* sm = h + 4;
    float tmn, tmx;
    std::memcpy(&tmn, sm + 5, 4);
    std::memcpy(&tmx, sm + 6, 4);
    info->n_grid = static_cast<int>(sm[0]);
    info->k_max = static_cast<int>(sm[1]);
    info->band_lo_min = static_cast<int>(sm[2]);
    info->spread_cells = static_cast<int>(sm[3]);
    info->band_width = static_cast<int>(sm[4]);
    info->tau_min = tmn;
    info->tau_max = tmx;
  }
  if (info && h[3]) info->proj_mode = 3;   // FP16x2 range exceeded: the projection ran on TF32x2
  if (h[0]) return fail(SKS_ERR_NONFINITE, "non-finite projection (NaN/Inf in x, y or an overflow)");
  if (h[2] & 1u)
    return fail(SKS_ERR_UNSUPPORTED, "NFFT grid beyond the built limit n = " + std::to_string(kNcap) +
                                         " (the kernel's spectrum is too wide for the data's range)");
  if (h[2] & 2u) return fail(SKS_ERR_UNSUPPORTED, "NDFT engine: Gaussian / Matern with at most 32 kept coefficients only");
  return SKS_OK;
}

// ---- CUDA-graph replay of whole calls (sks_options.graph): keyed by every argument of the call
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  sks_plan_info info{};
};
std::mutex g_graph_mu;
std::map<std::string, GraphEntry> g_graphs;

std::string graph_key(int dev, const void* a, const void* b, const void* c, const void* dd, const void* ws, size_t wsb,
                      int64_t N, int64_t M, int d, const sks_kernel& k, int P, uint64_t seed, int p0, int p1,
                      const Opts& o, cudaStream_t st) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%d|%p|%p|%p|%p|%p|%zu|%lld|%lld|%d|%d|%d|%.17g|%d|%llu|%d|%d|%.17g|%d|%d|%d|%d|%d|%p",
                dev, a, b, c, dd, ws, wsb, static_cast<long long>(N), static_cast<long long>(M), d, k.kind, k.matern_p,
                k.scale, P, static_cast<unsigned long long>(seed), p0, p1, o.eps, o.w, o.os, o.batch, o.engine, o.proj,
                static_cast<void*>(st));
  return buf;
}

}  // namespace

extern "C" {

const char* sks_version(void) { return "sks 0.2 (sm_100a)"; }

sks_status sks_release_caches(void) {
  int cur = 0;
  SKS_CUDA(cudaGetDevice(&cur));
  cudaError_t first = cudaSuccess;
  auto keep = [&](cudaError_t e) {
    if (first == cudaSuccess && e != cudaSuccess) first = e;
  };
  std::lock_guard<std::mutex> lg(g_graph_mu);   // (lock order: graphs, directions, plans -- as the calls take them)
  for (auto& kv : g_graphs) keep(cudaGraphExecDestroy(kv.second.exec));
  g_graphs.clear();
  std::lock_guard<std::mutex> ld(g_dir_mu);
  for (auto& kv : g_dirs) {
    keep(cudaSetDevice(std::get<0>(kv.first)));
    keep(cudaDeviceSynchronize());
    DirEntry& e = kv.second;
    keep(cudaFree(e.inv));
    keep(cudaFree(e.g3));
    keep(cudaFree(e.g32));
    keep(cudaFree(e.g16));
  }
  g_dirs.clear();
  std::lock_guard<std::mutex> lp(g_plan_mu);
  for (auto& kv : g_plans) {
    keep(cudaSetDevice(std::get<0>(kv.first)));
    keep(cudaDeviceSynchronize());
    keep(cudaFree(kv.second.phi2inv));
  }
  g_plans.clear();
  keep(cudaSetDevice(cur));
  if (first != cudaSuccess) return fail(SKS_ERR_CUDA, std::string("sks_release_caches: ") + cudaGetErrorString(first));
  return SKS_OK;
}

const char* sks_last_error(void) { return g_err.c_str(); }

sks_status sks_profile_enable(int32_t enable) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = enable != 0;
  return SKS_OK;
}

sks_status sks_profile_read(double* ms, int64_t* launches, int32_t n_slots) {
  if (!ms || !launches || n_slots < PS_N) return fail(SKS_ERR_INVALID, "need SKS_PROFILE_SLOTS slots");
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (auto& t : g_prof.pending) {
    const int slot = std::get<0>(t);
    cudaEvent_t a = std::get<1>(t), b = std::get<2>(t);
    float e = 0.f;
    SKS_CUDA(cudaEventSynchronize(b));
    SKS_CUDA(cudaEventElapsedTime(&e, a, b));
    g_prof.ms[slot] += e;
    g_prof.cnt[slot] += 1;
    g_prof.pool.push_back(a);
    g_prof.pool.push_back(b);
  }
  g_prof.pending.clear();
  for (int i = 0; i < PS_N; ++i) {
    ms[i] = g_prof.ms[i];
    launches[i] = g_prof.cnt[i];
    g_prof.ms[i] = 0.0;
    g_prof.cnt[i] = 0;
  }
  return SKS_OK;
}

const char* sks_profile_names(void) {
  return "split3,project,minmax,sp_hist,sp_part,sp_owner,sp_gather,reserved,plan,spread,fft_filter,eval,aux,"
         "ndft_spread,ndft_eval,sortsum";
}

sks_status sks_last_plan(sks_plan_info* info) {
  if (!info) return fail(SKS_ERR_INVALID, "info is NULL");
  *info = g_plan;
  return SKS_OK;
}

sks_status sks_sync_status(void* workspace, void* stream) {
  if (!workspace) return fail(SKS_ERR_INVALID, "workspace is NULL");
  return read_status(workspace, static_cast<cudaStream_t>(stream), &g_plan);
}

sks_status sks_directions(int32_t P, int32_t d, uint64_t seed, int32_t p_begin, int32_t p_end, float* g_out,
                          double* inv_norm_out) {
  if (P <= 0 || d <= 0 || p_begin < 0 || p_end > P || p_begin >= p_end) return fail(SKS_ERR_INVALID, "bad P/d/range");
  if (!g_out || !inv_norm_out) return fail(SKS_ERR_INVALID, "NULL output");
  sks::make_directions(P, d, seed, p_begin, p_end, g_out, inv_norm_out);
  return SKS_OK;
}

sks_status sks_fourier_coeffs(sks_kernel kernel, int32_t d, double tau, int32_t k0, int32_t k1, double* out) {
  sks_status s = check_kernel(kernel);
  if (s != SKS_OK) return s;
  if (kernel.kind == SKS_NEGDIST) return fail(SKS_ERR_UNSUPPORTED, "negdist has no Fourier path (Remark P:527-533)");
  if (d <= 0 || !(tau > 0) || k1 < k0 || !out) return fail(SKS_ERR_INVALID, "bad d/tau/range/out");
  sks::KernelModel km{kernel.kind, kernel.matern_p, kernel.scale, d};
  for (int32_t k = k0; k <= k1; ++k) out[k - k0] = sks::torus_coeff(km, tau, k < 0 ? -int64_t(k) : int64_t(k));
  return SKS_OK;
}

sks_status sks_workspace_size(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t P, int32_t p_begin,
                              int32_t p_end, const sks_options* opt, size_t* bytes) {
  sks_status s = validate_common(N, M, d, kernel, P, p_begin, p_end);
  if (s != SKS_OK) return s;
  Opts o;
  if ((s = resolve_opts(opt, &o)) != SKS_OK) return s;
  if (!bytes) return fail(SKS_ERR_INVALID, "bytes is NULL");
  const Path pt = path_of(kernel.kind);
  const bool fshape = fused_shape(N, d, pt, true, o.w) && o.engine != 2 && !o.det;
  const int batch = choose_batch(N, M, pt, p_end - p_begin, true, o.batch, d, o.proj, fshape);
  *bytes = make_layout(N, M, pt, batch, true, d, o.proj, fshape,
                       o.det ? det_groups(N, M, pt, p_end - p_begin, batch) : 0).total;
  return SKS_OK;
}

sks_status sks_sum(const float* x, int64_t N, const float* y, int64_t M, int32_t d, const float* w, sks_kernel kernel,
                   int32_t P, uint64_t seed, int32_t p_begin, int32_t p_end, float* s, void* workspace,
                   size_t workspace_bytes, const sks_options* opt, void* stream) {
  sks_status st = validate_common(N, M, d, kernel, P, p_begin, p_end);
  if (st != SKS_OK) return st;
  if (!x || !y || !w || !s) return fail(SKS_ERR_INVALID, "NULL x/y/w/s");
  Opts o;
  if ((st = resolve_opts(opt, &o)) != SKS_OK) return st;
  DirEntry dirs;
  if ((st = get_dirs(P, d, seed, p_begin, p_end, &dirs)) != SKS_OK) return st;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  Problem pr{N, M, d, kernel, p_end - p_begin, true};
  if (o.graph) {
    int dev = 0;
    SKS_CUDA(cudaGetDevice(&dev));
    const std::string key = graph_key(dev, x, y, w, s, workspace, workspace_bytes, N, M, d, kernel, P, seed, p_begin,
                                      p_end, o, cs);
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it == g_graphs.end()) {
      // first call with these arguments: run it eagerly (fills every cache and sets the kernels' attributes, so
      // the capture contains launches only), then capture the same launch sequence into a graph
      sks_plan_info info{};
      st = enqueue_call(pr, o, x, y, w, &dirs, nullptr, nullptr, s, nullptr, 1.0 / P, workspace, workspace_bytes, cs,
                        &info);
      if (st != SKS_OK) return st;
      g_plan = info;
      // capture on a private stream (the legacy default stream cannot be captured); replays go to `cs`
      cudaStream_t cap = nullptr;
      SKS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t graph = nullptr;
      SKS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      sks_plan_info info2{};
      const sks_status cst = enqueue_call(pr, o, x, y, w, &dirs, nullptr, nullptr, s, nullptr, 1.0 / P, workspace,
                                          workspace_bytes, cap, &info2);
      const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      if (cst != SKS_OK) return cst;
      if (ce != cudaSuccess) return fail(SKS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      GraphEntry ge;
      ge.info = info2;
      SKS_CUDA(cudaGraphInstantiate(&ge.exec, graph, 0));
      cudaGraphDestroy(graph);
      if (g_graphs.size() >= 64) {   // bounded: drop the whole cache (graphs are cheap to rebuild)
        for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second.exec);
        g_graphs.clear();
      }
      g_graphs.emplace(key, ge);
      return SKS_OK;
    }
    g_plan = it->second.info;
    SKS_CUDA(cudaGraphLaunch(it->second.exec, cs));
    return SKS_OK;
  }
  sks_plan_info info{};
  st = enqueue_call(pr, o, x, y, w, &dirs, nullptr, nullptr, s, nullptr, 1.0 / P, workspace, workspace_bytes, cs, &info);
  g_plan = info;
  if (st != SKS_OK || o.async) return st;
  return read_status(workspace, cs, &g_plan);
}

sks_status sks_workspace_size_host(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t P, int32_t p_begin,
                                   int32_t p_end, const sks_options* opt, size_t* bytes) {
  sks_status s = sks_workspace_size(N, M, d, kernel, P, p_begin, p_end, opt, bytes);
  if (s != SKS_OK) return s;
  *bytes += al(sizeof(float) * N * d) + al(sizeof(float) * M * d) + al(sizeof(float) * N) + al(sizeof(float) * M);
  return SKS_OK;
}

sks_status sks_sum_host(const float* x, int64_t N, const float* y, int64_t M, int32_t d, const float* w,
                        sks_kernel kernel, int32_t P, uint64_t seed, int32_t p_begin, int32_t p_end, float* s,
                        void* workspace, size_t workspace_bytes, const sks_options* opt, void* stream) {
  size_t need = 0;
  sks_status st = sks_workspace_size_host(N, M, d, kernel, P, p_begin, p_end, opt, &need);
  if (st != SKS_OK) return st;
  if (!x || !y || !w || !s) return fail(SKS_ERR_INVALID, "NULL x/y/w/s");
  if (!workspace || workspace_bytes < need) return fail(SKS_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return fail(SKS_ERR_INVALID, "workspace must be 256-byte aligned");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  // the compute workspace first (its status words at offset 0), then the device copies of x, y, w, s
  size_t inner = 0;
  if ((st = sks_workspace_size(N, M, d, kernel, P, p_begin, p_end, opt, &inner)) != SKS_OK) return st;
  char* ws = static_cast<char*>(workspace);
  float* dx = reinterpret_cast<float*>(ws + al(inner));
  float* dy = reinterpret_cast<float*>(reinterpret_cast<char*>(dx) + al(sizeof(float) * N * d));
  float* dw = reinterpret_cast<float*>(reinterpret_cast<char*>(dy) + al(sizeof(float) * M * d));
  float* ds = reinterpret_cast<float*>(reinterpret_cast<char*>(dw) + al(sizeof(float) * N));
  SKS_CUDA(cudaMemcpyAsync(dx, x, sizeof(float) * N * d, cudaMemcpyHostToDevice, cs));
  SKS_CUDA(cudaMemcpyAsync(dy, y, sizeof(float) * M * d, cudaMemcpyHostToDevice, cs));
  SKS_CUDA(cudaMemcpyAsync(dw, w, sizeof(float) * N, cudaMemcpyHostToDevice, cs));
  sks_options o{};
  if (opt) o = *opt;
  o.async = 1;   // one synchronisation below covers the result copy and the status
  o.graph = 0;
  st = sks_sum(dx, N, dy, M, d, dw, kernel, P, seed, p_begin, p_end, ds, ws, inner, &o, stream);
  if (st != SKS_OK) return st;
  SKS_CUDA(cudaMemcpyAsync(s, ds, sizeof(float) * M, cudaMemcpyDeviceToHost, cs));
  return read_status(ws, cs, &g_plan);
}

sks_status sks_project(const float* pts, int64_t n, int32_t d, int32_t P, uint64_t seed, int32_t p_begin,
                       int32_t p_end, float* z, const sks_options* opt, void* stream) {
  if (!pts || !z || n <= 0 || d <= 0) return fail(SKS_ERR_INVALID, "bad pts/z/n/d");
  if (n > INT32_MAX) return fail(SKS_ERR_INVALID, "n must be < 2^31");
  if (P <= 0 || p_begin < 0 || p_end > P || p_begin >= p_end) return fail(SKS_ERR_INVALID, "bad slice range");
  Opts o;
  sks_status st = resolve_opts(opt, &o);
  if (st != SKS_OK) return st;
  DirEntry dirs;
  if ((st = get_dirs(P, d, seed, p_begin, p_end, &dirs)) != SKS_OK) return st;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int np = p_end - p_begin;
  // ranges / flag / split scratch are not needed by the caller: a small per-thread scratch (allocated on
  // first use, grown on demand; this entry point is a test/inspection aid, not the hot path)
  static thread_local unsigned* scratch = nullptr;
  static thread_local size_t scratch_bytes = 0;
  const ProjMode pm = proj_mode_call(d, o.proj, pts, n, pts, 0);
  const bool tc = pm == PM_BF16X3;
  const size_t need = al(sizeof(unsigned) * 4 * np + 16) +
                      (tc ? al(sizeof(uint16_t) * 3 * sks::proj_tc_dpad(d) * n) + al(sks::proj_tc_part_bytes(np)) : 0);
  if (scratch_bytes < need) {
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    SKS_CUDA(cudaMalloc(&scratch, need));
    scratch_bytes = need;
  }
  unsigned* mm = scratch;
  int* flag = reinterpret_cast<int*>(scratch + 4 * np);
  SKS_CUDA(cudaMemsetAsync(flag, 0, 16, cs));   // flag and the FP16x2 sampled max
  SKS_CUDA(sks::launch_init_minmax(mm, np, cs));
  if (tc) {
    char* xs3 = reinterpret_cast<char*>(scratch) + al(sizeof(unsigned) * 4 * np + 16);
    char* part = xs3 + al(sizeof(uint16_t) * 3 * sks::proj_tc_dpad(d) * n);
    SKS_CUDA(sks::launch_split3(pts, n, pts, 0, d, xs3, cs));
    SKS_CUDA(sks::launch_project_tc(xs3, n, n, d, dirs.g3, np, dirs.inv, z, n, mm, flag, part, cs));
  } else if (pm == PM_FP16X2) {   // (+ the TF32x2 rerun, predicated on a point outside the fp16 range)
    unsigned* f16 = reinterpret_cast<unsigned*>(flag);
    SKS_CUDA(sks::launch_project_f16(pts, n, pts, 0, d, dirs.g16, np, dirs.inv, z, n, mm, flag, f16 + 1, cs));
    SKS_CUDA(sks::launch_rerun_prep(f16, mm, np, cs));
    SKS_CUDA(sks::launch_project_tf32(pts, n, pts, 0, d, dirs.g32, np, dirs.inv, z, n, mm, flag, f16 + 3, cs));
  } else {
    SKS_CUDA(sks::launch_project_tf32(pts, n, pts, 0, d, dirs.g32, np, dirs.inv, z, n, mm, flag, nullptr, cs));
  }
  return SKS_OK;
}

sks_status sks_workspace_size_1d(int64_t N, int64_t M, int32_t d, sks_kernel kernel, int32_t n_slices,
                                 const sks_options* opt, size_t* bytes) {
  sks_status s = validate_common(N, M, d, kernel, n_slices, 0, n_slices);
  if (s != SKS_OK) return s;
  Opts o;
  if ((s = resolve_opts(opt, &o)) != SKS_OK) return s;
  if (!bytes) return fail(SKS_ERR_INVALID, "bytes is NULL");
  const Path pt = path_of(kernel.kind);
  const int batch = choose_batch(N, M, pt, n_slices, false, o.batch, d, o.proj, false);
  *bytes = make_layout(N, M, pt, batch, false, d, o.proj, false).total;
  return SKS_OK;
}

sks_status sks_sum_1d(const float* zx, const float* zy, const float* w, int64_t N, int64_t M, int32_t n_slices,
                      int32_t d, sks_kernel kernel, float* t, void* workspace, size_t workspace_bytes,
                      const sks_options* opt, void* stream) {
  sks_status st = validate_common(N, M, d, kernel, n_slices, 0, n_slices);
  if (st != SKS_OK) return st;
  if (!zx || !zy || !w || !t) return fail(SKS_ERR_INVALID, "NULL zx/zy/w/t");
  Opts o;
  if ((st = resolve_opts(opt, &o)) != SKS_OK) return st;
  Problem pr{N, M, d, kernel, n_slices, false};
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  sks_plan_info info{};
  st = enqueue_call(pr, o, nullptr, nullptr, w, nullptr, zx, zy, nullptr, t, 1.0, workspace, workspace_bytes, cs, &info);
  g_plan = info;
  if (st != SKS_OK || o.async) return st;
  return read_status(workspace, cs, &g_plan);
}

}  // extern "C"
