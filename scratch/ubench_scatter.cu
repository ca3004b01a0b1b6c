// Microbenchmark: costs of the un-permutation options of the sort path on B200
//   (1) scattered fp64 RED to global (s64 accumulate), (2) scattered fp32 stores to global,
//   (3) scattered fp32 stores to DSMEM (cluster of C), (4) scattered fp32 stores to local smem,
//   (5) coalesced float2 stores to global, (6) random 8-byte LDS, (7) cp.async.bulk smem->dsmem copy.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void k_red64(int iters, double* arr, uint32_t mask) {
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); atomicAdd(arr + (s & mask), 1.0); }
}
__global__ void k_red32(int iters, float* arr, uint32_t mask) {
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); atomicAdd(arr + (s & mask), 1.0f); }
}
__global__ void k_st32(int iters, float* arr, uint32_t mask) {
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); arr[s & mask] = (float)it; }
}
__global__ void k_st64co(int iters, float2* arr, uint32_t mask) {
  const uint32_t base = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) arr[(base + it * gridDim.x * blockDim.x) & mask] = make_float2(it, it);
}
template <int C>
__global__ void k_dsm_st(int iters, float* out) {
  extern __shared__ float sh[];   // 16384 floats
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sh[i] = 0.f;
  cl.sync();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = hsh(s + it);
    float* r = cl.map_shared_rank(sh, (s >> 20) % C);
    r[s & 16383] = (float)it;
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}
template <int C>
__global__ void k_dsm_red(int iters, float* out) {
  extern __shared__ float sh[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sh[i] = 0.f;
  cl.sync();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = hsh(s + it);
    float* r = cl.map_shared_rank(sh, (s >> 20) % C);
    atomicAdd(r + (s & 16383), 1.0f);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}
__global__ void k_smem_st(int iters, float* out) {
  extern __shared__ float sh[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); sh[s & 16383] = (float)it; }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}
__global__ void k_smem_ld64(int iters, float* out) {
  extern __shared__ float2 sh2[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sh2[i] = make_float2(i, i);
  __syncthreads();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); const float2 v = sh2[s & 8191]; acc += v.x * v.y; }
  if (acc == 12345.f) out[0] = acc;
}
// gather: scattered 8-byte global loads (L2-resident table)
__global__ void k_gather64(int iters, const float2* arr, uint32_t mask, float* out) {
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) { s = hsh(s + it); const float2 v = __ldcg(arr + (s & mask)); acc += v.x; }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  float* out; CK(cudaMalloc(&out, 1 << 24));
  double* arr; CK(cudaMalloc(&arr, size_t(8) << 22)); CK(cudaMemset(arr, 0, size_t(8) << 22));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = 148 * 2, threads = 1024, iters = 256;
  double nops = (double)blocks * threads * iters;
  float ms;
  auto run = [&](const char* name, auto launch) {
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-48s %8.3f ms %8.2f Gop/s  %.3f cyc/op/SM @1.95GHz\n", name, ms, nops / ms / 1e6, (ms * 1e-3 * 1.95e9 * 148) / nops);
    return 0;
  };
  // 1e5-entry (800 KB) target like s64 for cfg2
  run("RED.f64 global, 128K addr (1 MB)", [&] { k_red64<<<blocks, threads>>>(iters, arr, (1u << 17) - 1); });
  run("RED.f64 global, 4M addr (32 MB)", [&] { k_red64<<<blocks, threads>>>(iters, arr, (1u << 22) - 1); });
  run("RED.f32 global, 128K addr", [&] { k_red32<<<blocks, threads>>>(iters, (float*)arr, (1u << 17) - 1); });
  run("ST.f32 global scattered, 128K addr", [&] { k_st32<<<blocks, threads>>>(iters, (float*)arr, (1u << 17) - 1); });
  run("ST.f32 global scattered, 8M addr", [&] { k_st32<<<blocks, threads>>>(iters, (float*)arr, (1u << 23) - 1); });
  run("ST.64 global coalesced, 4M addr", [&] { k_st64co<<<blocks, threads>>>(iters, (float2*)arr, (1u << 22) - 1); });
  run("LD.64 global gather, 128K addr (1 MB)", [&] { k_gather64<<<blocks, threads>>>(iters, (const float2*)arr, (1u << 17) - 1, out); });
  run("LD.64 global gather, 4M addr (32 MB)", [&] { k_gather64<<<blocks, threads>>>(iters, (const float2*)arr, (1u << 22) - 1, out); });
  CK(cudaFuncSetAttribute(k_smem_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  run("STS.32 scattered local smem", [&] { k_smem_st<<<blocks, threads, 65536>>>(iters, out); });
  CK(cudaFuncSetAttribute(k_smem_ld64, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  run("LDS.64 random local smem", [&] { k_smem_ld64<<<blocks, threads, 65536>>>(iters, out); });
  auto dsm = [&](auto kern, int C, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(C * (C > 8 ? 8 : 148 / C)); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 65536;
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = C; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    double save = nops; nops = (double)cfg.gridDim.x * threads * iters;
    run(name, [&] { cudaLaunchKernelEx(&cfg, kern, iters, out); });
    nops = save;
    return 0;
  };
  dsm(k_dsm_st<2>, 2, "ST.f32 DSMEM scattered, cluster 2");
  dsm(k_dsm_st<4>, 4, "ST.f32 DSMEM scattered, cluster 4");
  dsm(k_dsm_st<8>, 8, "ST.f32 DSMEM scattered, cluster 8");
  dsm(k_dsm_red<4>, 4, "RED.f32 DSMEM scattered, cluster 4");
  dsm(k_dsm_red<8>, 8, "RED.f32 DSMEM scattered, cluster 8");
  CK(cudaGetLastError());
  return 0;
}
